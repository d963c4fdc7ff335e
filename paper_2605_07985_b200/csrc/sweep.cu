// K5 — fused sweep -> fit (replaces sweep + oracle_latency
// + fit for signatures whose measurements come from the analytical model:
// SPEC.md:466-484, D3 :515, fit :556-564).
//
// One thread per signature.  The thread enumerates the signature's sweep grid
// in the order of profiler.sweep_points (App. A.5), evaluates the roofline
// latency model of profiler.op_cost / oracle_latency in registers — in the
// same floating-point operation order as the Python host model, so every y is
// bit-identical — and feeds the points straight into the moment accumulators.
// The solve and the training-MAPE pass regenerate the points instead of
// reading them back: no measurement ever touches HBM (the host sweep + K2
// path moves 12-20 B per point twice).  Optionally the generated (x, y) are
// written out for verification.
#include "attn_moments.cuh"
#include "common.cuh"

namespace dooly {

constexpr double SWEEP_DROP_TOL = 1e-9;

__device__ __forceinline__ double rcp64s(double y) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y));
  double e = fma(-y, r, 1.0);
  r = fma(r, e, r);
  e = fma(-y, r, 1.0);
  return fma(r, e, r);
}

struct SweepPoint {
  uint32_t x[3];
  double y;
};

// (flops, bytes) of one op instance, Python operator order of profiler.op_cost.
__device__ __forceinline__ void op_cost(const dooly_sweep_desc& d, int64_t t, int64_t r,
                                        int64_t c, bool prefill, double& flops, double& nbytes) {
  const int64_t db = d.dtype_bytes;
  switch (d.op) {
    case DOOLY_OP_LINEAR: {
      const int64_t k = d.dim[0], n = d.dim[1];
      const int64_t m = d.feature == DOOLY_FEAT_NUM_SEQS ? r : t;
      flops = mul(mul(mul(2.0, (double)m), (double)k), (double)n);
      nbytes = (double)((m * k + k * n + m * n) * db);
      return;
    }
    case DOOLY_OP_EMBEDDING:
      flops = 0.0;
      nbytes = (double)(2 * t * d.dim[0] * db + 4 * t);
      return;
    case DOOLY_OP_RMSNORM:
      flops = mul(mul(4.0, (double)t), (double)d.dim[0]);
      nbytes = (double)((2 * t * d.dim[0] + d.dim[0]) * db);
      return;
    case DOOLY_OP_ROTARY: {
      const int64_t w = d.dim[0];
      flops = mul(mul(3.0, (double)t), (double)w);
      nbytes = (double)(2 * t * w * db);
      return;
    }
    case DOOLY_OP_ACT_MUL: {
      const int64_t i2 = d.dim[0];
      flops = mul(mul(2.0, (double)t), (double)i2);
      nbytes = (double)((t * i2 + t * i2 / 2) * db);
      return;
    }
    case DOOLY_OP_TOPK: {
      const int64_t e = d.dim[0];
      flops = mul(mul(5.0, (double)t), (double)e);
      nbytes = (double)(t * e * (db + 8));
      return;
    }
    case DOOLY_OP_MOE: {
      const int64_t e = d.dim[0], i2 = d.dim[1], h = d.dim[2], k = d.dim[3];
      const int64_t touched = e < t * k ? e : t * k;
      flops = mul(mul(mul(mul(2.0, (double)t), (double)k), (double)(i2 + i2 / 2)), (double)h);
      nbytes = (double)((touched * (i2 + i2 / 2) * h + 2 * t * h) * db);
      return;
    }
    case DOOLY_OP_ATTENTION: {
      const double hq = (double)d.dim[0], hd = (double)d.dim[1], hkv = (double)d.dim[2];
      int64_t ce = c;
      if (d.window > 0 && d.window < ce) ce = d.window;
      const double q = prefill ? __ddiv_rn((double)t, (double)r) : 1.0;
      const double ctx = add((double)ce, q);
      const double rr = (double)r;
      flops = mul(mul(mul(mul(mul(4.0, hq), hd), rr), q), ctx);
      const double a = mul(mul(mul(mul(rr, ctx), 2.0), hkv), hd);
      const double b = mul(mul(mul((double)(2 * r), q), hq), hd);
      nbytes = mul((double)db, add(a, b));
      return;
    }
    default:  // reshape / unknown: overhead only
      flops = 0.0;
      nbytes = 0.0;
  }
}

__device__ __forceinline__ double latency(const dooly_sweep_desc& d, const dooly_sweep_grid& g,
                                          double flops, double nbytes, bool prefill) {
  const double m = d.feature == DOOLY_FEAT_ATTN ? (prefill ? d.mult[0] : d.mult[1]) : d.mult[0];
  const double a = __ddiv_rn(flops, g.peak_flops), b = __ddiv_rn(nbytes, g.mem_bw);
  return add(g.overhead, mul(m, b > a ? b : a));
}

// Enumerate the signature's points (profiler.sweep_points order) and call f.
template <typename F>
__device__ __forceinline__ void for_each_point(const dooly_sweep_desc& d, const dooly_sweep_grid& g,
                                               F&& f) {
  const int64_t cap_t = g.chunk < d.max_context ? g.chunk : d.max_context;
  if (d.feature == DOOLY_FEAT_NUM_TOKS) {
    for (int i = 0; i < g.n_tok; ++i) {
      const int64_t t = g.tok[i];
      if (t > cap_t) continue;
      double fl, nb;
      op_cost(d, t, 1, 0, false, fl, nb);
      SweepPoint p{{(uint32_t)t, 0u, 0u}, latency(d, g, fl, nb, false)};
      f(p);
    }
    return;
  }
  if (d.feature == DOOLY_FEAT_NUM_SEQS) {
    for (int j = 0; j < g.n_req; ++j) {
      const int64_t r = g.req[j];
      if (r > g.max_batch) continue;
      double fl, nb;
      op_cost(d, 1, r, 0, false, fl, nb);
      SweepPoint p{{(uint32_t)r, 0u, 0u}, latency(d, g, fl, nb, false)};
      f(p);
    }
    return;
  }
  const int64_t W = d.window > 0 ? d.window : 0;
  for (int i = 0; i < g.n_tok; ++i) {  // prefill points
    const int64_t t = g.tok[i];
    if (t > cap_t) continue;
    for (int j = 0; j < g.n_req; ++j) {
      const int64_t r = g.req[j];
      if (r > g.max_batch || t < r) continue;
      for (int k = 0; k < g.n_kv; ++k) {
        const int64_t c = g.kv[k];
        if (c + (t + r - 1) / r > d.max_context) continue;
        double fl, nb;
        op_cost(d, t, r, c, true, fl, nb);
        const int64_t ce = W && W < c ? W : c;
        SweepPoint p{{(uint32_t)t, (uint32_t)r, (uint32_t)(r * ce)}, latency(d, g, fl, nb, true)};
        f(p);
      }
    }
  }
  for (int j = 0; j < g.n_req; ++j) {  // decode points
    const int64_t r = g.req[j];
    if (r > g.max_batch) continue;
    for (int k = 0; k < g.n_kv; ++k) {
      const int64_t c = g.kv[k];
      if (c + 1 > d.max_context) continue;
      double fl, nb;
      op_cost(d, r, r, c, false, fl, nb);
      const int64_t ce = W && W < c ? W : c;
      SweepPoint p{{0u, (uint32_t)r, (uint32_t)(r * ce)}, latency(d, g, fl, nb, false)};
      f(p);
    }
  }
}

// Serial Cholesky-with-drop solve of G c = b (lower triangle of G used).
template <int NC>
__device__ __forceinline__ void chol_solve(double (*G)[NC], const double* b, double* c) {
  double rd[NC], z[NC];
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    const double gjj = G[j][j];
    double d2 = gjj;
#pragma unroll
    for (int k = 0; k < j; ++k) d2 = fma(-G[j][k], G[j][k], d2);
    const bool keep = d2 > SWEEP_DROP_TOL * gjj;
    const double dd = keep ? sqrt(d2) : 0.0;
    rd[j] = keep ? rcp64s(dd) : 0.0;
    G[j][j] = dd;
#pragma unroll
    for (int i = j + 1; i < NC; ++i) {
      double t = G[i][j];
#pragma unroll
      for (int k = 0; k < j; ++k) t = fma(-G[i][k], G[j][k], t);
      G[i][j] = t * rd[j];
    }
  }
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    double t = b[j];
#pragma unroll
    for (int k = 0; k < j; ++k) t = fma(-G[j][k], z[k], t);
    z[j] = t * rd[j];
  }
#pragma unroll
  for (int j = NC - 1; j >= 0; --j) {
    double t = z[j];
#pragma unroll
    for (int k = j + 1; k < NC; ++k) t = fma(-G[k][j], c[k], t);
    c[j] = t * rd[j];
  }
}

__device__ __forceinline__ double u2d_s(uint32_t x) {
  return __hiloint2double(0x43300000, (int)x) - 4503599627370496.0;
}

template <int KIND>
__global__ void __launch_bounds__(128) profile_fit_kernel(
    const dooly_sweep_desc* __restrict__ descs, int64_t n_sig, const dooly_sweep_grid grid,
    void* __restrict__ table, double* __restrict__ fit_err, uint8_t* __restrict__ status,
    uint32_t* __restrict__ out_x, double* __restrict__ out_y, const int64_t* __restrict__ out_off,
    int64_t out_n) {
  constexpr int P = KIND == DOOLY_KIND_ATTN ? 3 : 1;
  constexpr int NC = KIND == DOOLY_KIND_ATTN ? 10 : 2;
  constexpr int NEED = KIND == DOOLY_KIND_ATTN ? 11 : 4;
  constexpr int NACC = KIND == DOOLY_KIND_ATTN ? 44 : 4;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n_sig;
       s += (int64_t)gridDim.x * blockDim.x) {
    const dooly_sweep_desc d = descs[s];
    double acc[NACC];
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = 0.0;
    uint32_t lo[P], hi[P];
#pragma unroll
    for (int k = 0; k < P; ++k) {
      lo[k] = 0xFFFFFFFFu;
      hi[k] = 0u;
    }
    int64_t n = 0;
    const int64_t o = out_off != nullptr ? out_off[s] : 0;
    for_each_point(d, grid, [&](const SweepPoint& p) {
      if (out_x != nullptr) {
#pragma unroll
        for (int k = 0; k < P; ++k) out_x[k * out_n + o + n] = p.x[k];
        out_y[o + n] = p.y;
      }
      double v[P];
#pragma unroll
      for (int k = 0; k < P; ++k) {
        v[k] = u2d_s(p.x[k]);
        lo[k] = min(lo[k], p.x[k]);
        hi[k] = max(hi[k], p.x[k]);
      }
      if constexpr (KIND == DOOLY_KIND_ATTN) {
        attn_accumulate(v[0], v[1], v[2], p.y, acc);
      } else {
        acc[0] += v[0];
        acc[1] = fma(v[0], v[0], acc[1]);
        acc[2] += p.y;
        acc[3] = fma(p.y, v[0], acc[3]);
      }
      ++n;
    });
    if (n < NEED) {
      if constexpr (KIND == DOOLY_KIND_AFFINE) {
        dooly_affine_row* row = static_cast<dooly_affine_row*>(table) + s;
        row->c0 = row->c1 = row->inv_scale = nan64();
        row->lo = 0xFFFFFFFFu;
        row->hi = 0;
      } else {
        dooly_attn_row* row = static_cast<dooly_attn_row*>(table) + s;
        for (int i = 0; i < 10; ++i) row->c[i] = nan64();
        for (int k = 0; k < 3; ++k) {
          row->inv_scale[k] = nan64();
          row->lo[k] = 0xFFFFFFFFu;
          row->hi[k] = 0;
        }
      }
      fit_err[s] = nan64();
      status[s] = DOOLY_FIT_INSUFFICIENT;
      continue;
    }
    double inv[P];
#pragma unroll
    for (int k = 0; k < P; ++k) inv[k] = hi[k] > 0 ? 1.0 / (double)hi[k] : 1.0;
    double G[NC][NC], b[NC], c[NC];
    if constexpr (KIND == DOOLY_KIND_ATTN) {
      double sc[35], msc[35];
      attn_monomials(inv[0], inv[1], inv[2], sc);
      msc[0] = (double)n;
#pragma unroll
      for (int m = 1; m < 35; ++m) msc[m] = acc[m - 1] * sc[m];
      attn_gram(msc, G);
#pragma unroll
      for (int i = 0; i < NC; ++i) b[i] = acc[34 + i] * sc[attn_colmon(i)];
    } else {
      G[0][0] = (double)n;
      G[1][0] = acc[0] * inv[0];
      G[1][1] = acc[1] * inv[0] * inv[0];
      b[0] = acc[2];
      b[1] = acc[3] * inv[0];
    }
    chol_solve<NC>(G, b, c);
    // pass 2: regenerate the points for the training MAPE
    double err = 0.0;
    for_each_point(d, grid, [&](const SweepPoint& p) {
      double v[P];
#pragma unroll
      for (int k = 0; k < P; ++k) v[k] = u2d_s(p.x[k]) * inv[k];
      double pr;
      if constexpr (KIND == DOOLY_KIND_ATTN) {
        pr = fma(c[1], v[0], c[0]);
        pr = fma(c[2], v[1], pr);
        pr = fma(c[3], v[2], pr);
        pr = fma(c[4], v[0] * v[0], pr);
        pr = fma(c[5], v[1] * v[1], pr);
        pr = fma(c[6], v[2] * v[2], pr);
        pr = fma(c[7], v[0] * v[1], pr);
        pr = fma(c[8], v[0] * v[2], pr);
        pr = fma(c[9], v[1] * v[2], pr);
      } else {
        pr = fma(c[1], v[0], c[0]);
      }
      pr = fmax(pr, DOOLY_CLAMP_FLOOR);
      err = fma(fabs(pr - p.y), rcp64s(p.y), err);
    });
    fit_err[s] = err / (double)n;
    status[s] = DOOLY_FIT_OK;
    if constexpr (KIND == DOOLY_KIND_AFFINE) {
      dooly_affine_row* row = static_cast<dooly_affine_row*>(table) + s;
      row->c0 = c[0];
      row->c1 = c[1];
      row->inv_scale = inv[0];
      row->lo = lo[0];
      row->hi = hi[0];
    } else {
      dooly_attn_row* row = static_cast<dooly_attn_row*>(table) + s;
      for (int i = 0; i < 10; ++i) row->c[i] = c[i];
      for (int k = 0; k < 3; ++k) {
        row->inv_scale[k] = inv[k];
        row->lo[k] = lo[k];
        row->hi[k] = hi[k];
      }
    }
  }
}

cudaError_t launch_profile_fit(int kind, const dooly_sweep_desc* descs, int64_t n_sig,
                               const dooly_sweep_grid* grid, void* table, double* fit_err,
                               uint8_t* status, uint32_t* out_x, double* out_y,
                               const int64_t* out_off, int64_t out_n, cudaStream_t stream,
                               int n_sm) {
  if (n_sig == 0) return cudaSuccess;
  int64_t blocks = (n_sig + 127) / 128;
  const int64_t cap = (int64_t)n_sm * 16;
  if (blocks > cap) blocks = cap;
  if (kind == DOOLY_KIND_AFFINE)
    profile_fit_kernel<DOOLY_KIND_AFFINE><<<(unsigned)blocks, 128, 0, stream>>>(
        descs, n_sig, *grid, table, fit_err, status, out_x, out_y, out_off, out_n);
  else
    profile_fit_kernel<DOOLY_KIND_ATTN><<<(unsigned)blocks, 128, 0, stream>>>(
        descs, n_sig, *grid, table, fit_err, status, out_x, out_y, out_off, out_n);
  return cudaGetLastError();
}

}  // namespace dooly
