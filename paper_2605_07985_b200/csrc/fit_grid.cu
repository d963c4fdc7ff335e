// K2g — shared-grid fit (dooly_fit_grid): the fit of SPEC.md:556-564 for the
// common case where every signature of a batch was swept over the SAME points
// (one sweep grid per model/backend; the C5 scale sweep).
//
// With a shared design matrix M (n_pts x p) the normal-equation Gram M^T M,
// its Cholesky-with-drop factor, the solve matrix W (c = W b), the scaling
// (inv = 1/max x), the training box and the scaled feature planes
// f_k(p) = RN(x_k(p) * inv_k) are the same for every signature, so they are
// computed ONCE (fit_grid_prep_kernel, one CTA, into the workspace).  Per
// signature only X^T y remains:
//   pass 1  b = M^T y          (13 FP64 per point for the 10-column design)
//   solve   c = W b            (lanes 0..p-1, one coefficient each)
//   pass 2  training MAPE      (9-FMA regrouped polynomial + 1-Newton reciprocal)
// versus ~95 FP64 instructions per point for the per-signature Gram path
// (fit.cu).
//
// Four kernels share this contract:
//   fit_grid_db_kernel    (affine default) the warp kernel with the y loads of
//                         the next YS steps in flight while the current YS
//                         steps are evaluated (register double buffer).
//   fit_grid_warp_kernel  (attention default) one warp per signature, no shared-memory
//                         stage, no CTA barrier: y streamed from HBM with
//                         L2::evict_last, 8 steps in flight per lane, re-read
//                         from L2 in pass 2; f planes from L1.
//   fit_grid_stage_kernel (DOOLY_FIT_GRID_KERNEL=stage) R signatures per CTA
//                         staged in shared memory by 1-D TMA.
//   fit_grid_kernel       (unaligned or n_pts % 4 != 0) the same with direct
//                         global loads.
//
// Result contract: identical to dooly_fit with pt_off[s] = s * n_pts and x
// repeated per signature — coefficients within 1e-9 normwise, fit_err within
// the MAPE bound (tests/test_gpu_fit_grid.py), same row layout and statuses.
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "common.cuh"

namespace dooly {

constexpr double kGridDropTol = 1e-9;  // App. A.7, same rule as fit.cu
constexpr int kGT = 256;
constexpr int kGW = kGT / 32;

template <int KIND>
struct GridTraits;
template <>
struct GridTraits<DOOLY_KIND_AFFINE> {
  static constexpr int P = 1, NC = 2, NEED = 4, R = 8, RS = 3;
};
template <>
struct GridTraits<DOOLY_KIND_ATTN> {
  static constexpr int P = 3, NC = 10, NEED = 11, R = 4, RS = 3;
};
constexpr size_t kGridStageMax = 96 * 1024;  // y bytes staged per CTA (2 CTAs/SM)

struct GridFactor {
  double L[10][10];  // lower Cholesky factor; dropped columns are zero
  double W[10][10];  // c = W b: the forward+backward solve with drop applied to e_i
  double rd[10];     // 1 / L[j][j], 0 for a dropped column
  double inv[3];
  uint32_t lo[3], hi[3];
  int32_t ok;        // n_pts >= need
  int32_t grp4;      // attention: x0 and x1 constant on every aligned group of 4 points
  // packed 96-B serving form (attention): bit-field layout of the box, as
  // dooly_attn_pack derives it (widths from the largest fitted hi)
  uint32_t pk_s1, pk_s2;  // bit offsets of the second and third box fields
  int32_t pk_ok;          // the three widths fit in 64 bits
  int32_t f3p128;         // attention: x2 periodic with a period dividing 128 points
};

// Epilogue destinations: the peer tables of the fused all-gather and,
// optionally, the packed 96-B attention rows (dooly_fit_grid_packed).
struct GridOut : dooly_grid_peers {
  uint8_t* packed;   // header row + one row per signature, or null
};

static size_t grid_factor_bytes() { return (sizeof(GridFactor) + 255) & ~(size_t)255; }

__device__ __forceinline__ double g_u2d(uint32_t x) {
  return __hiloint2double(0x43300000, (int)x) - 4503599627370496.0;
}

// x * inv in one rounding: 2^52 + x is exact (x < 2^32) and nbias = -2^52 * inv
// is a power-of-two scaling of inv, so the fused product-sum rounds the exact
// x * inv once — bit-identical to g_u2d(x) * inv in one FP64 instruction.
__device__ __forceinline__ double g_scale(uint32_t x, double inv, double nbias) {
  return fma(__hiloint2double(0x43300000, (int)x), inv, nbias);
}

__device__ __forceinline__ double g_rcp(double y) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y));
  double e = fma(-y, r, 1.0);
  r = fma(r, e, r);
  e = fma(-y, r, 1.0);
  return fma(r, e, r);
}

// One Newton step on the hardware estimate: ~2^-44 relative, ample for the
// training-MAPE diagnostic (1e-9 contract).
__device__ __forceinline__ double g_rcp1(double y) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y));
  return fma(r, fma(-y, r, 1.0), r);
}

template <typename T>
__device__ __forceinline__ T g_warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}

// Design columns in eval order (common.cuh eval_attn): [1,f1,f2,f3,f1²,f2²,f3²,f1f2,f1f3,f2f3].
template <int KIND>
__device__ __forceinline__ void grid_monomials(const uint32_t* xs, const double* inv, double* m) {
  if constexpr (KIND == DOOLY_KIND_AFFINE) {
    m[0] = 1.0;
    m[1] = g_u2d(xs[0]) * inv[0];
  } else {
    const double f1 = g_u2d(xs[0]) * inv[0], f2 = g_u2d(xs[1]) * inv[1],
                 f3 = g_u2d(xs[2]) * inv[2];
    m[0] = 1.0;
    m[1] = f1;
    m[2] = f2;
    m[3] = f3;
    m[4] = f1 * f1;
    m[5] = f2 * f2;
    m[6] = f3 * f3;
    m[7] = f1 * f2;
    m[8] = f1 * f3;
    m[9] = f2 * f3;
  }
}

// Training-MAPE prediction from the scaled features only (pass 2): the same
// polynomial as the design row, regrouped so it needs 9 FMAs and no monomials
//   c0 + f1(c1 + c4 f1 + c7 f2 + c8 f3) + f2(c2 + c5 f2 + c9 f3) + f3(c3 + c6 f3).
// fit_err is a diagnostic held to 1e-9 relative, not the bit-exact predict
// contract, so the regrouping is allowed here (and only here).
template <int KIND>
__device__ __forceinline__ double grid_horner(const double* c, const double* f) {
  if constexpr (KIND == DOOLY_KIND_AFFINE) {
    return fma(c[1], f[0], c[0]);
  } else {
    const double t1 = fma(c[8], f[2], fma(c[7], f[1], fma(c[4], f[0], c[1])));
    const double t2 = fma(c[9], f[2], fma(c[5], f[1], c[2]));
    const double t3 = fma(c[6], f[2], c[3]);
    return fma(f[0], t1, fma(f[1], t2, fma(f[2], t3, c[0])));
  }
}

template <int KIND>
__device__ __forceinline__ void grid_features(const uint32_t* xs, const double* inv,
                                              const double* nb, double* f) {
  constexpr int P = KIND == DOOLY_KIND_AFFINE ? 1 : 3;
#pragma unroll
  for (int k = 0; k < P; ++k) f[k] = g_scale(xs[k], inv[k], nb[k]);
}

// One CTA: box, scaling, Gram of the shared design, Cholesky with drop.
template <int KIND>
__global__ void __launch_bounds__(kGT) fit_grid_prep_kernel(const uint32_t* __restrict__ x,
                                                            int64_t n_pts, GridFactor* gf,
                                                            double* __restrict__ fplanes,
                                                            uint8_t* packed, int64_t n_rows) {
  using T = GridTraits<KIND>;
  constexpr int P = T::P, NC = T::NC, NT = NC * (NC + 1) / 2;
  __shared__ uint32_t smn[kGW][3], smx[kGW][3];
  __shared__ double sg[kGW][NT];
  __shared__ double G[NC][NC];
  __shared__ double sinv[3];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  uint32_t mn[P], mx[P];
#pragma unroll
  for (int k = 0; k < P; ++k) {
    mn[k] = 0xFFFFFFFFu;
    mx[k] = 0u;
  }
  for (int64_t p = tid; p < n_pts; p += kGT)
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const uint32_t v = x[k * n_pts + p];
      mn[k] = min(mn[k], v);
      mx[k] = max(mx[k], v);
    }
#pragma unroll
  for (int k = 0; k < P; ++k) {
    const uint32_t a = __reduce_min_sync(0xFFFFFFFFu, mn[k]);
    const uint32_t b = __reduce_max_sync(0xFFFFFFFFu, mx[k]);
    if (lane == 0) {
      smn[wid][k] = a;
      smx[wid][k] = b;
    }
  }
  __syncthreads();
  if (tid < P) {
    uint32_t a = 0xFFFFFFFFu, b = 0u;
    for (int w = 0; w < kGW; ++w) {
      a = min(a, smn[w][tid]);
      b = max(b, smx[w][tid]);
    }
    gf->lo[tid] = a;
    gf->hi[tid] = b;
    const double iv = b > 0 ? 1.0 / (double)b : 1.0;  // IEEE division, as the oracle
    gf->inv[tid] = iv;
    sinv[tid] = iv;
  }
  __syncthreads();
  double inv[P];
#pragma unroll
  for (int k = 0; k < P; ++k) inv[k] = sinv[k];
  for (int64_t p = tid; p < n_pts; p += kGT)
#pragma unroll
    for (int k = 0; k < P; ++k)
      fplanes[k * n_pts + p] = g_scale(x[k * n_pts + p], inv[k], -4503599627370496.0 * inv[k]);
  if (KIND == DOOLY_KIND_ATTN && n_pts % 4 == 0) {   // 16-B aligned only then
    // group plane for the grouped passes: (f1, f2) of each aligned 4-point group
    double2* gpl = reinterpret_cast<double2*>(fplanes + 3 * n_pts);
    for (int64_t g = tid; g < n_pts / 4; g += kGT)
      gpl[g] = make_double2(g_scale(x[4 * g], inv[0], -4503599627370496.0 * inv[0]),
                            g_scale(x[n_pts + 4 * g], inv[1], -4503599627370496.0 * inv[1]));
  }
  double acc[NT];
#pragma unroll
  for (int i = 0; i < NT; ++i) acc[i] = 0.0;
  for (int64_t p = tid; p < n_pts; p += kGT) {
    uint32_t xs[P];
#pragma unroll
    for (int k = 0; k < P; ++k) xs[k] = x[k * n_pts + p];
    double m[NC];
    grid_monomials<KIND>(xs, inv, m);
    int t = 0;
#pragma unroll
    for (int i = 0; i < NC; ++i)
#pragma unroll
      for (int j = i; j < NC; ++j) acc[t] = fma(m[i], m[j], acc[t]), ++t;
  }
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    const double v = g_warp_sum(acc[i]);
    if (lane == 0) sg[wid][i] = v;
  }
  __syncthreads();
  if (tid < NT) {
    int i = 0, t = tid;
    while (t >= NC - i) {
      t -= NC - i;
      ++i;
    }
    const int j = i + t;
    double v = 0.0;
    for (int w = 0; w < kGW; ++w) v += sg[w][tid];
    G[i][j] = v;
    G[j][i] = v;
  }
  // Sweep grids nest the kv axis innermost: when every
  // aligned group of 4 points shares prefill_toks and batch, pass 1 of the warp
  // kernel factors those two features out of the group's sums.
  int grp4 = 0;
  if constexpr (KIND == DOOLY_KIND_ATTN) {
    grp4 = n_pts % 4 == 0 ? 1 : 0;
    for (int64_t g = tid; grp4 && g < n_pts / 4; g += kGT) {
      const uint32_t* a = x + 4 * g;
      const uint32_t* b = x + n_pts + 4 * g;
      grp4 = (a[1] == a[0] && a[2] == a[0] && a[3] == a[0] && b[1] == b[0] && b[2] == b[0] &&
              b[3] == b[0]) ? 1 : 0;
    }
  }
  grp4 = __syncthreads_and(grp4);
  // ... and when the kv axis repeats with a period dividing 128 points (the C5
  // 16-value kv axis does), a warp-kernel lane sees the same four f3 values at
  // every step (its points are 4 lane + 128 t): it keeps them in registers
  int f3p = 0;
  if constexpr (KIND == DOOLY_KIND_ATTN) {
    f3p = n_pts % 128 == 0 ? 1 : 0;
    const uint32_t* x2 = x + 2 * n_pts;
    for (int64_t q = 128 + tid; f3p && q < n_pts; q += kGT) f3p = x2[q] == x2[q & 127] ? 1 : 0;
  }
  f3p = __syncthreads_and(f3p);
  if (tid == 0) {
    gf->grp4 = grp4;
    gf->f3p128 = f3p;
    double diag[NC];
    for (int j = 0; j < NC; ++j) diag[j] = G[j][j];
    for (int j = 0; j < NC; ++j) {
      const double piv = G[j][j];
      const bool keep = piv > kGridDropTol * diag[j];
      const double d = keep ? sqrt(piv) : 0.0;
      const double id = keep ? 1.0 / d : 0.0;
      gf->rd[j] = id;
      for (int i = 0; i < NC; ++i) gf->L[i][j] = i < j ? 0.0 : (i == j ? d : G[i][j] * id);
      for (int k = j + 1; k < NC; ++k)
        for (int i = k; i < NC; ++i) G[i][k] = fma(-gf->L[i][j], gf->L[k][j], G[i][k]);
    }
    for (int i = NC; i < 10; ++i) gf->rd[i] = 0.0;
    // W = the solve applied to the unit vectors, so per signature c = W b is
    // NC independent dot products instead of two dependent triangular sweeps.
    for (int e = 0; e < NC; ++e) {
      double z[NC], c[NC];
      for (int j = 0; j < NC; ++j) {
        double t = j == e ? 1.0 : 0.0;
        for (int i = 0; i < j; ++i) t = fma(-gf->L[j][i], z[i], t);
        z[j] = t * gf->rd[j];
      }
      for (int j = NC - 1; j >= 0; --j) {
        double t = z[j];
        for (int i = j + 1; i < NC; ++i) t = fma(-gf->L[i][j], c[i], t);
        c[j] = t * gf->rd[j];
      }
      for (int j = 0; j < NC; ++j) gf->W[j][e] = c[j];
    }
    gf->ok = n_pts >= T::NEED ? 1 : 0;
    if constexpr (KIND == DOOLY_KIND_ATTN) {
      // packed-form field widths from the largest fitted hi (every fitted row
      // carries the grid's box), as dooly_attn_pack's scan would find them
      uint32_t w[3], mh[3];
      for (int k = 0; k < 3; ++k) {
        mh[k] = gf->ok ? gf->hi[k] : 0u;
        w[k] = max(1, 32 - __clz((int)mh[k]));
      }
      gf->pk_s1 = w[0];
      gf->pk_s2 = w[0] + w[1];
      gf->pk_ok = (w[0] + w[1] + w[2] <= 64) ? 1 : 0;
      if (packed != nullptr) {
        dooly_attn_pack_header h;
        memset(&h, 0, sizeof(h));
        h.magic = DOOLY_PACK_MAGIC;
        h.ok = gf->pk_ok ? 1u : 0u;   // inv = 1/hi by construction: no bad_inv rows
        for (int k = 0; k < 3; ++k) {
          h.width[k] = w[k];
          h.max_hi[k] = mh[k];
        }
        h.n_sig = n_rows;
        *reinterpret_cast<dooly_attn_pack_header*>(packed) = h;
      }
    }
  }
}

// Row emission.  Rows go to the local table at global row pe.row0 + s and,
// for the fused fit + all-gather (dooly_fit_grid_bcast), to every peer rank's
// table at the same row over peer memory (NVLink P2P stores): the regressor
// all-gather of SURVEY §8(e) happens in the fit's own epilogue.  A row is
// assembled in registers and written as 16-B stores.
template <int KIND>
struct RowBuf {
  static constexpr int N2 = KIND == DOOLY_KIND_AFFINE ? 2 : 8;  // double2 per row
  double2 v[N2];
};

template <int KIND>
__device__ __forceinline__ RowBuf<KIND> make_row(const double* c, const double* inv,
                                                 const uint32_t* lo, const uint32_t* hi) {
  RowBuf<KIND> r;
  if constexpr (KIND == DOOLY_KIND_AFFINE) {
    r.v[0] = make_double2(c[0], c[1]);
    r.v[1] = make_double2(inv[0], __longlong_as_double((long long)(((uint64_t)hi[0] << 32) | lo[0])));
  } else {
#pragma unroll
    for (int i = 0; i < 5; ++i) r.v[i] = make_double2(c[2 * i], c[2 * i + 1]);
    r.v[5] = make_double2(inv[0], inv[1]);
    r.v[6] = make_double2(inv[2], __longlong_as_double((long long)(((uint64_t)lo[1] << 32) | lo[0])));
    r.v[7] = make_double2(__longlong_as_double((long long)(((uint64_t)hi[0] << 32) | lo[2])),
                          __longlong_as_double((long long)(((uint64_t)hi[2] << 32) | hi[1])));
  }
  return r;
}

template <int KIND>
__device__ __forceinline__ void put_row(void* table, int64_t row, const RowBuf<KIND>& r) {
  double2* d = reinterpret_cast<double2*>(table) + row * RowBuf<KIND>::N2;
#pragma unroll
  for (int i = 0; i < RowBuf<KIND>::N2; ++i) d[i] = r.v[i];
}

template <int KIND>
__device__ __forceinline__ void emit_row(const GridOut& pe, const GridFactor* gf, void* table,
                                         double* fit_err, uint8_t* status, int64_t s,
                                         const RowBuf<KIND>& r, double err, uint8_t st) {
  const int64_t g = pe.row0 + s;
  put_row<KIND>(table, g, r);
  fit_err[g] = err;
  status[g] = st;
  if constexpr (KIND == DOOLY_KIND_ATTN) {
    if (pe.packed != nullptr) {
      // the 96-B serving row, exactly as dooly_attn_pack writes it: the
      // folded coefficients, then the box bit-packed with the table's field widths
      const uint64_t w6 = (uint64_t)__double_as_longlong(r.v[6].y);
      const uint64_t w7a = (uint64_t)__double_as_longlong(r.v[7].x);
      const uint64_t w7b = (uint64_t)__double_as_longlong(r.v[7].y);
      const uint32_t lo0 = (uint32_t)w6, lo1 = (uint32_t)(w6 >> 32), lo2 = (uint32_t)w7a;
      const uint32_t hi0 = (uint32_t)(w7a >> 32), hi1 = (uint32_t)w7b, hi2 = (uint32_t)(w7b >> 32);
      uint64_t lb = ~0ull, hb = 0ull;
      if (lo0 <= hi0 && gf->pk_ok) {
        lb = (uint64_t)lo0 | ((uint64_t)lo1 << gf->pk_s1) | ((uint64_t)lo2 << gf->pk_s2);
        hb = (uint64_t)hi0 | ((uint64_t)hi1 << gf->pk_s1) | ((uint64_t)hi2 << gf->pk_s2);
      }
      double c[10], inv[3] = {r.v[5].x, r.v[5].y, r.v[6].x}, w[12];
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        c[2 * i] = r.v[i].x;
        c[2 * i + 1] = r.v[i].y;
      }
      fold_row96(c, inv, lb, hb, w);
      double2* o = reinterpret_cast<double2*>(pe.packed + 96 * (1 + g));
#pragma unroll
      for (int i = 0; i < 6; ++i) o[i] = make_double2(w[2 * i], w[2 * i + 1]);
    }
  }
  for (int p = 0; p < pe.n_peers; ++p) {
    put_row<KIND>(pe.table[p], g, r);
    pe.fit_err[p][g] = err;
    pe.status[p][g] = st;
  }
  if (pe.n_peers > 0) __threadfence_system();  // peer stores ordered before the arrival signal
}

template <int KIND>
__device__ void write_unfitted_grid(const GridOut& pe, const GridFactor* gf, void* table,
                                    int64_t s, double* fit_err, uint8_t* status) {
  double c[10], inv[3];
  uint32_t lo[3], hi[3];
  for (int i = 0; i < 10; ++i) c[i] = nan64();
  for (int k = 0; k < 3; ++k) {
    inv[k] = nan64();
    lo[k] = 0xFFFFFFFFu;
    hi[k] = 0;
  }
  emit_row<KIND>(pe, gf, table, fit_err, status, s, make_row<KIND>(c, inv, lo, hi), nan64(),
                 DOOLY_FIT_INSUFFICIENT);
}

template <int KIND>
__global__ void __launch_bounds__(kGT, 2) fit_grid_kernel(
    const uint32_t* __restrict__ x, int64_t n_pts, const double* __restrict__ y, int64_t n_sig,
    const GridFactor* __restrict__ gf, void* __restrict__ table, double* __restrict__ fit_err,
    uint8_t* __restrict__ status, const GridOut pe) {
  using T = GridTraits<KIND>;
  constexpr int P = T::P, NC = T::NC, R = T::R;
  __shared__ double sL[NC][NC], srd[NC], sinv[P];
  __shared__ uint32_t slo[P], shi[P];
  __shared__ double part[kGW][R * NC];
  __shared__ double scoef[R][NC];
  __shared__ double serr[kGW][R];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int t = tid; t < NC * NC; t += kGT) sL[t / NC][t % NC] = gf->L[t / NC][t % NC];
  if (tid < NC) srd[tid] = gf->rd[tid];
  if (tid < P) {
    sinv[tid] = gf->inv[tid];
    slo[tid] = gf->lo[tid];
    shi[tid] = gf->hi[tid];
  }
  const bool ok = gf->ok != 0;
  __syncthreads();
  double inv[P];
#pragma unroll
  for (int k = 0; k < P; ++k) inv[k] = sinv[k];
  const int64_t n_groups = (n_sig + R - 1) / R;
  for (int64_t g = blockIdx.x; g < n_groups; g += gridDim.x) {
    const int64_t s0 = g * R;
    const int nr = (int)min((int64_t)R, n_sig - s0);
    if (!ok) {
      if (tid < nr) write_unfitted_grid<KIND>(pe, gf, table, s0 + tid, fit_err, status);
      continue;
    }
    const double* yg = y + s0 * n_pts;
    // ---- pass 1: b = M^T y for R signatures
    double acc[R][NC];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int k = 0; k < NC; ++k) acc[r][k] = 0.0;
    for (int64_t p = tid; p < n_pts; p += kGT) {
      uint32_t xs[P];
#pragma unroll
      for (int k = 0; k < P; ++k) xs[k] = __ldg(x + k * n_pts + p);
      double yv[R];
#pragma unroll
      for (int r = 0; r < R; ++r) yv[r] = r < nr ? yg[r * n_pts + p] : 0.0;
      double m[NC];
      grid_monomials<KIND>(xs, inv, m);
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int k = 0; k < NC; ++k) acc[r][k] = fma(yv[r], m[k], acc[r][k]);
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        const double v = g_warp_sum(acc[r][k]);
        if (lane == 0) part[wid][r * NC + k] = v;
      }
    __syncthreads();
    // ---- solve with the shared factor (thread r owns signature r)
    if (tid < nr) {
      double z[NC];
#pragma unroll
      for (int j = 0; j < NC; ++j) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < kGW; ++w) t += part[w][tid * NC + j];
#pragma unroll
        for (int i = 0; i < j; ++i) t = fma(-sL[j][i], z[i], t);
        z[j] = t * srd[j];
      }
#pragma unroll
      for (int j = NC - 1; j >= 0; --j) {
        double t = z[j];
#pragma unroll
        for (int i = j + 1; i < NC; ++i) t = fma(-sL[i][j], scoef[tid][i], t);
        scoef[tid][j] = t * srd[j];
      }
    }
    __syncthreads();
    // ---- pass 2: training MAPE (y rows re-read, normally from L2)
    double c[R][NC], err[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      err[r] = 0.0;
#pragma unroll
      for (int k = 0; k < NC; ++k) c[r][k] = scoef[r][k];
    }
    for (int64_t p = tid; p < n_pts; p += kGT) {
      uint32_t xs[P];
#pragma unroll
      for (int k = 0; k < P; ++k) xs[k] = __ldg(x + k * n_pts + p);
      double yv[R];
#pragma unroll
      for (int r = 0; r < R; ++r) yv[r] = r < nr ? yg[r * n_pts + p] : 1.0;
      double m[NC];
      grid_monomials<KIND>(xs, inv, m);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double pr = c[r][0];
#pragma unroll
        for (int k = 1; k < NC; ++k) pr = fma(c[r][k], m[k], pr);
        pr = fmax(pr, DOOLY_CLAMP_FLOOR);
        err[r] = fma(fabs(pr - yv[r]), g_rcp(yv[r]), err[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double v = g_warp_sum(err[r]);
      if (lane == 0) serr[wid][r] = v;
    }
    __syncthreads();
    if (tid < nr) {
      double e = 0.0;
#pragma unroll
      for (int w = 0; w < kGW; ++w) e += serr[w][tid];
      emit_row<KIND>(pe, gf, table, fit_err, status, s0 + tid,
                     make_row<KIND>(scoef[tid], sinv, slo, shi), e / (double)n_pts,
                     DOOLY_FIT_OK);
    }
    __syncthreads();
  }
}

// ---- staged variant: the R signatures' y rows are bulk-copied (1-D TMA) into
// shared memory in two point-halves, so both passes read smem and y crosses
// HBM exactly once (8 B/point).  The next group's first half is copied in as
// soon as pass 2 has released it.
__device__ __forceinline__ uint32_t g_smem(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void g_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          g_smem(dst)),
      "l"(src), "r"(bytes), "r"(g_smem(bar))
      : "memory");
}
__device__ __forceinline__ void g_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(g_smem(bar)), "r"(parity)
        : "memory");
}

template <int KIND>
__global__ void __launch_bounds__(kGT, 2) fit_grid_stage_kernel(
    const uint32_t* __restrict__ x, int64_t n_pts, const double* __restrict__ y, int64_t n_sig,
    const GridFactor* __restrict__ gf, void* __restrict__ table, double* __restrict__ fit_err,
    uint8_t* __restrict__ status, const GridOut pe) {
  using T = GridTraits<KIND>;
  constexpr int P = T::P, NC = T::NC, R = T::RS;
  extern __shared__ __align__(128) unsigned char gdyn[];
  double* stage = reinterpret_cast<double*>(gdyn);  // [R][n_pts]
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ double sW[NC][NC], sb[R * NC], sinv[P];
  __shared__ uint32_t slo[P], shi[P];
  __shared__ double part[kGW][R * NC];
  __shared__ double scoef[R][NC];
  __shared__ double serr[kGW][R];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t half = n_pts / 2;  // n_pts % 4 == 0 (launcher)
  const int n = (int)n_pts;        // stage <= 96 KB, so n_pts <= 12288
  const int64_t n_groups = (n_sig + R - 1) / R;
  for (int t = tid; t < NC * NC; t += kGT) sW[t / NC][t % NC] = gf->W[t / NC][t % NC];
  if (tid < P) {
    sinv[tid] = gf->inv[tid];
    slo[tid] = gf->lo[tid];
    shi[tid] = gf->hi[tid];
  }
  const bool ok = gf->ok != 0;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(g_smem(&bar[0])));
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(g_smem(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t g, int c) {  // thread 0: half c of group g
    const int64_t s0 = g * R;
    const int nr = (int)min((int64_t)R, n_sig - s0);
    const uint32_t bytes = (uint32_t)(half * 8);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(g_smem(&bar[c])),
                 "r"(bytes * nr)
                 : "memory");
    for (int r = 0; r < nr; ++r)
      g_bulk(stage + r * n_pts + c * half, y + (s0 + r) * n_pts + c * half, bytes, &bar[c]);
  };
  double inv[P], nb[P];
#pragma unroll
  for (int k = 0; k < P; ++k) inv[k] = sinv[k], nb[k] = -4503599627370496.0 * sinv[k];
  if (!ok) {
    for (int64_t g = blockIdx.x; g < n_groups; g += gridDim.x) {
      const int nr = (int)min((int64_t)R, n_sig - g * R);
      if (tid < nr) write_unfitted_grid<KIND>(pe, gf, table, g * R + tid, fit_err, status);
    }
    return;
  }
  if (tid == 0 && blockIdx.x < n_groups) {
    issue(blockIdx.x, 0);
    issue(blockIdx.x, 1);
  }
  uint32_t par[2] = {0u, 0u};
  for (int64_t g = blockIdx.x; g < n_groups; g += gridDim.x) {
    const int64_t s0 = g * R;
    const int nr = (int)min((int64_t)R, n_sig - s0);
    const int64_t gn = g + gridDim.x;
    double acc[R][NC];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int k = 0; k < NC; ++k) acc[r][k] = 0.0;
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      g_wait(&bar[c], par[c]);
      par[c] ^= 1u;
      // two consecutive points per thread: 8-B x loads, 16-B y loads, 32-bit indices
      for (int p = (int)(c * half) + 2 * tid; p < (int)((c + 1) * half); p += 2 * kGT) {
        uint32_t xa[P], xb[P];
#pragma unroll
        for (int k = 0; k < P; ++k) {
          const uint2 v = __ldg(reinterpret_cast<const uint2*>(x + k * n + p));
          xa[k] = v.x;
          xb[k] = v.y;
        }
        double ma[NC], mb[NC];
        grid_monomials<KIND>(xa, inv, ma);
        grid_monomials<KIND>(xb, inv, mb);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double2 yv =
              r < nr ? *reinterpret_cast<const double2*>(stage + r * n + p) : make_double2(0.0, 0.0);
#pragma unroll
          for (int k = 0; k < NC; ++k) acc[r][k] = fma(yv.y, mb[k], fma(yv.x, ma[k], acc[r][k]));
        }
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        const double v = g_warp_sum(acc[r][k]);
        if (lane == 0) part[wid][r * NC + k] = v;
      }
    __syncthreads();
    if (tid < R * NC) {  // b = sum of the warp partials
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < kGW; ++w) t += part[w][tid];
      sb[tid] = t;
    }
    __syncthreads();
    if (tid < nr * NC) {  // c = W b, one coefficient per thread
      const int r = tid / NC, j = tid - r * NC;
      double c = 0.0;
#pragma unroll
      for (int i = 0; i < NC; ++i) c = fma(sW[j][i], sb[r * NC + i], c);
      scoef[r][j] = c;
    }
    __syncthreads();
    double cf[R][NC], err[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      err[r] = 0.0;
#pragma unroll
      for (int k = 0; k < NC; ++k) cf[r][k] = scoef[r][k];
    }
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      for (int p = (int)(c * half) + 2 * tid; p < (int)((c + 1) * half); p += 2 * kGT) {
        uint32_t xa[P], xb[P];
#pragma unroll
        for (int k = 0; k < P; ++k) {
          const uint2 v = __ldg(reinterpret_cast<const uint2*>(x + k * n + p));
          xa[k] = v.x;
          xb[k] = v.y;
        }
        double fa[P], fb[P];
        grid_features<KIND>(xa, inv, nb, fa);
        grid_features<KIND>(xb, inv, nb, fb);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double2 yv =
              r < nr ? *reinterpret_cast<const double2*>(stage + r * n + p) : make_double2(1.0, 1.0);
          double pa = grid_horner<KIND>(cf[r], fa), pb = grid_horner<KIND>(cf[r], fb);
          pa = fmax(pa, DOOLY_CLAMP_FLOOR);
          pb = fmax(pb, DOOLY_CLAMP_FLOOR);
          err[r] = fma(fabs(pa - yv.x), g_rcp1(yv.x), err[r]);
          err[r] = fma(fabs(pb - yv.y), g_rcp1(yv.y), err[r]);
        }
      }
      if (c == 0) {
        __syncthreads();  // half 0 released: stream in the next group's first half
        if (tid == 0 && gn < n_groups) issue(gn, 0);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double v = g_warp_sum(err[r]);
      if (lane == 0) serr[wid][r] = v;
    }
    __syncthreads();  // half 1 released
    if (tid == 0 && gn < n_groups) issue(gn, 1);
    if (tid < nr) {
      double e = 0.0;
#pragma unroll
      for (int w = 0; w < kGW; ++w) e += serr[w][tid];
      emit_row<KIND>(pe, gf, table, fit_err, status, s0 + tid,
                     make_row<KIND>(scoef[tid], sinv, slo, shi), e / (double)n_pts,
                     DOOLY_FIT_OK);
    }
    __syncthreads();  // scoef / part reused by the next group
  }
}

// Grouped attention steps (the 4 points of a lane share f1 = u1 and f2 = u2,
// prep's grp4): pass 1 as kv sums times the group's f1/f2 monomials (7.25 FP64
// per point instead of 13), pass 2 with the f1/f2 terms folded per group into
// p = A + f3 (B + c6 f3) (8.75 instead of 14).
__device__ __forceinline__ void grid_g1_step(const double4& yv, const double4& f3, double u1,
                                             double u2, double* acc) {
  const double yy[4] = {yv.x, yv.y, yv.z, yv.w};
  const double ff[4] = {f3.x, f3.y, f3.z, f3.w};
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double y3 = yy[j] * ff[j];
    s0 += yy[j];
    s1 += y3;
    s2 = fma(y3, ff[j], s2);
  }
  const double u11 = u1 * u1, u22 = u2 * u2, u12 = u1 * u2;
  acc[0] += s0;
  acc[1] = fma(u1, s0, acc[1]);
  acc[2] = fma(u2, s0, acc[2]);
  acc[3] += s1;
  acc[4] = fma(u11, s0, acc[4]);
  acc[5] = fma(u22, s0, acc[5]);
  acc[6] += s2;
  acc[7] = fma(u12, s0, acc[7]);
  acc[8] = fma(u1, s1, acc[8]);
  acc[9] = fma(u2, s1, acc[9]);
}

// Pass 1 when a lane also sees the same four f3 values at every step (f3p128):
// f3 leaves the per-point work entirely.  Per lane position j the step sums
// T_j = sum y, U1_j = sum u1 y, U2_j = sum u2 y (3 FP64 per point), and the
// three moments quadratic in (u1, u2) take the group sum S0 (3 + 3 + 3 per
// group): 5.25 FP64 per point instead of 7.25.  grid_r1_fold forms the ten
// moments from them with the lane's f3 quad once per signature.
struct GridR1 {
  double T[4], U1[4], U2[4], Q[3];
};

__device__ __forceinline__ void grid_r1_step(const double4& yv, double u1, double u2, GridR1& r) {
  const double yy[4] = {yv.x, yv.y, yv.z, yv.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    r.T[j] += yy[j];
    r.U1[j] = fma(u1, yy[j], r.U1[j]);
    r.U2[j] = fma(u2, yy[j], r.U2[j]);
  }
  const double s0 = (yy[0] + yy[1]) + (yy[2] + yy[3]);
  r.Q[0] = fma(u1 * u1, s0, r.Q[0]);
  r.Q[1] = fma(u2 * u2, s0, r.Q[1]);
  r.Q[2] = fma(u1 * u2, s0, r.Q[2]);
}

__device__ __forceinline__ void grid_r1_fold(const GridR1& r, const double4& f3, double* acc) {
  const double ff[4] = {f3.x, f3.y, f3.z, f3.w};
  acc[0] = (r.T[0] + r.T[1]) + (r.T[2] + r.T[3]);
  acc[1] = (r.U1[0] + r.U1[1]) + (r.U1[2] + r.U1[3]);
  acc[2] = (r.U2[0] + r.U2[1]) + (r.U2[2] + r.U2[3]);
  acc[4] = r.Q[0];
  acc[5] = r.Q[1];
  acc[7] = r.Q[2];
  acc[3] = acc[6] = acc[8] = acc[9] = 0.0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double t3 = r.T[j] * ff[j];
    acc[3] += t3;
    acc[6] = fma(t3, ff[j], acc[6]);
    acc[8] = fma(r.U1[j], ff[j], acc[8]);
    acc[9] = fma(r.U2[j], ff[j], acc[9]);
  }
}

__device__ __forceinline__ void grid_g2_step(const double4& yv, const double4& f3, double u1,
                                             double u2, const double* c, double& err) {
  const double t1 = fma(c[7], u2, fma(c[4], u1, c[1]));
  const double t2 = fma(c[5], u2, c[2]);
  const double A = fma(u1, t1, fma(u2, t2, c[0]));
  const double B = fma(c[9], u2, fma(c[8], u1, c[3]));
  const double yy[4] = {yv.x, yv.y, yv.z, yv.w};
  const double ff[4] = {f3.x, f3.y, f3.z, f3.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double pr = fmax(fma(ff[j], fma(c[6], ff[j], B), A), DOOLY_CLAMP_FLOOR);
    err = fma(fabs(pr - yy[j]), g_rcp1(yy[j]), err);
  }
}

// ---- warp-per-signature variant (no shared-memory stage, no CTA barriers).
// One warp owns one signature at a time: pass 1 streams its y row from HBM
// tagged L2::evict_last, the warp reduces b with shuffles, lanes 0..NC-1 form
// c = W b and broadcast it, and pass 2 re-reads the row — an L2 hit, because
// the launch keeps (warps in flight x 8 B x n_pts) well inside L2 — tagged
// evict_first.  x (the shared grid) is read through L1, which this kernel
// leaves entirely to it.  y crosses HBM once; there is no stage to fill or
// drain, so every warp streams independently.
__device__ __forceinline__ double4 g_ld_y(const double* p, bool keep) {
  double4 v;
  if (keep)
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_last.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
                 : "l"(p));
  else
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
                 : "l"(p));
  return v;
}

// Feature planes: read-only, shared by every warp, kept in L1.
__device__ __forceinline__ double4 g_ld_f(const double* p) {
  double4 v;
  asm("ld.global.nc.L1::evict_last.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
      : "l"(p));
  return v;
}

// ---- per-warp bulk-copy ring (attention, f3-periodic grouped grids).
// ncu of the warp kernel: y latency binds it (long_scoreboard 2.75 of 7.1
// cycles per issue, DRAM 62%, FP64 pipe 54%) because the y loads in flight
// live in registers (8 steps x 8 registers per lane) and the register file
// caps residency at 16 warps/SM.  Here every warp streams its OWN signatures
// through a private NS-stage shared-memory ring filled by 1-D TMA
// (cp.async.bulk, mbarrier complete_tx): lane 0 keeps NS chunks of CHB bytes
// in flight without a register, the lanes read each chunk with two
// conflict-free LDS.128 per step (the halves of a lane's 32 B swapped on
// lanes with bit 2 set, and the lane's f3 quad permuted to match), and the
// ring runs on across the pass and signature boundaries, so the next
// signature's pass 1 streams in while this one is solved and emitted.  No CTA
// barrier, no cross-warp traffic: the arithmetic is the warp kernel's
// (grid_r1_step / grid_g2_step).  Pass 2's chunks come from L2 (pass 1
// copies with an evict_last policy, pass 2 with evict_first).
constexpr int kRingPts = 512;  // n_pts must be a multiple (every ring variant's chunk divides it)

template <int NS, int CHB, int MINB>
__global__ void __launch_bounds__(256, MINB) fit_grid_ring_kernel(
    const double* __restrict__ fpl, int64_t n_pts, const double* __restrict__ y, int64_t n_sig,
    const GridFactor* __restrict__ gf, void* __restrict__ table, double* __restrict__ fit_err,
    uint8_t* __restrict__ status, const GridOut pe) {
  constexpr int KIND = DOOLY_KIND_ATTN, NC = 10, STEPS = CHB / 1024;
  static_assert(CHB % 1024 == 0 && (kRingPts * 8) % CHB == 0, "chunk = whole 128-point steps");
  extern __shared__ __align__(128) unsigned char rdyn[];
  __shared__ double sW[NC][NC];
  __shared__ double sinv[3];
  __shared__ uint32_t slo[3], shi[3];
  __shared__ __align__(8) uint64_t rbar[8][NS];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int n = (int)n_pts;
  if (!(gf->ok && gf->grp4 && gf->f3p128 && n % kRingPts == 0)) return;  // warp kernel's case
  for (int t = tid; t < NC * NC; t += blockDim.x) sW[t / NC][t % NC] = gf->W[t / NC][t % NC];
  if (tid < 3) {
    sinv[tid] = gf->inv[tid];
    slo[tid] = gf->lo[tid];
    shi[tid] = gf->hi[tid];
  }
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NS; ++i)
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(g_smem(&rbar[wid][i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned char* ring = rdyn + (size_t)wid * NS * CHB;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + tid) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nch = n * 8 / CHB;  // chunks per pass
  const int64_t per_sig = 2 * (int64_t)nch;
  const int64_t my_sigs = warp < n_sig ? (n_sig - 1 - warp) / n_warps + 1 : 0;
  const int64_t total = my_sigs * per_sig;
  uint64_t pol_keep = 0, pol_first = 0;
  if (lane == 0) {
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
  }
  // lane 0's issue cursor (incremental: no 64-bit division per chunk):
  // signature is_s, chunk is_w of its 2 nch, stage is_st; left = chunks to issue
  int64_t is_s = warp, left = total;
  int is_w = 0, is_st = 0;
  auto issue = [&]() {
    const bool p1 = is_w < nch;
    const double* src = y + is_s * (int64_t)n + (int64_t)(p1 ? is_w : is_w - nch) * (CHB / 8);
    uint64_t* bar = &rbar[wid][is_st];
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(g_smem(bar)), "r"(CHB)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(g_smem(ring + is_st * CHB)),
        "l"(src), "r"(CHB), "r"(g_smem(bar)), "l"(p1 ? pol_keep : pol_first)
        : "memory");
    if (++is_w == 2 * nch) {
      is_w = 0;
      is_s += n_warps;
    }
    is_st = is_st + 1 == NS ? 0 : is_st + 1;
    --left;
  };
  if (lane == 0)
    for (int i = 0; i < NS && left > 0; ++i) issue();
  const int h = (lane >> 2) & 1;  // bank swizzle of the two 16-B halves
  const double4 f3 = g_ld_f(fpl + 2 * n + 4 * lane);
  const double4 f3q = h ? make_double4(f3.z, f3.w, f3.x, f3.y) : f3;
  const double2* gpl = reinterpret_cast<const double2*>(fpl + 3 * n);
  // consume cursor: stage c_st, its phase parity c_ph
  int c_st = 0;
  uint32_t c_ph = 0;
  // chunk w of the current pass: wait for it, evaluate its STEPS steps,
  // release the stage to the chunk NS ahead
  auto consume = [&](int w, auto&& step) {
    g_wait(&rbar[wid][c_st], c_ph);
    const unsigned char* base = ring + c_st * CHB + 32 * lane;
#pragma unroll
    for (int t = 0; t < STEPS; ++t) {
      const double2 a = *reinterpret_cast<const double2*>(base + 1024 * t + 16 * h);
      const double2 b = *reinterpret_cast<const double2*>(base + 1024 * t + 16 * (1 - h));
      const double2 u = __ldg(gpl + ((w * (CHB / 8) + 128 * t + 4 * lane) >> 2));
      step(make_double4(a.x, a.y, b.x, b.y), u);
    }
    __syncwarp();  // every lane's reads of the stage precede the refill
    if (lane == 0 && left > 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue();
    }
    if (++c_st == NS) {
      c_st = 0;
      c_ph ^= 1u;
    }
  };
  for (int64_t si = 0; si < my_sigs; ++si) {
    const int64_t s = warp + si * n_warps;
    GridR1 r1;
#pragma unroll
    for (int j = 0; j < 4; ++j) r1.T[j] = r1.U1[j] = r1.U2[j] = 0.0;
    r1.Q[0] = r1.Q[1] = r1.Q[2] = 0.0;
    for (int w = 0; w < nch; ++w)
      consume(w, [&](const double4& yv, const double2& u) { grid_r1_step(yv, u.x, u.y, r1); });
    double c[NC];
    {
      double acc[NC];
      grid_r1_fold(r1, f3q, acc);
#pragma unroll
      for (int i = 0; i < NC; ++i) acc[i] = g_warp_sum(acc[i]);
      double cj = 0.0;
      if (lane < NC) {
#pragma unroll
        for (int i = 0; i < NC; ++i) cj = fma(sW[lane][i], acc[i], cj);
      }
#pragma unroll
      for (int i = 0; i < NC; ++i) c[i] = __shfl_sync(0xFFFFFFFFu, cj, i);
    }
    double err = 0.0;
    for (int w = 0; w < nch; ++w)
      consume(w, [&](const double4& yv, const double2& u) {
        grid_g2_step(yv, f3q, u.x, u.y, c, err);
      });
    err = g_warp_sum(err);
    if (lane == 0)
      emit_row<KIND>(pe, gf, table, fit_err, status, s, make_row<KIND>(c, sinv, slo, shi),
                     err / (double)n, DOOLY_FIT_OK);
  }
}

#ifndef FG_WARP_MINB
#define FG_WARP_MINB 2  // CTAs per SM the warp kernel's registers are sized for
#endif
#ifndef FG_WARP_YS
#define FG_WARP_YS 8    // y steps (4 points per lane each) issued ahead of their math
#endif
template <int KIND>
__global__ void __launch_bounds__(256, FG_WARP_MINB) fit_grid_warp_kernel(
    const double* __restrict__ fpl, int64_t n_pts, const double* __restrict__ y, int64_t n_sig,
    const GridFactor* __restrict__ gf, void* __restrict__ table, double* __restrict__ fit_err,
    uint8_t* __restrict__ status, const GridOut pe, int allow_factor, int su_groups) {
  using T = GridTraits<KIND>;
  constexpr int P = T::P, NC = T::NC;
  // the (f1, f2) group plane staged in shared memory (su_groups > 0): the
  // grouped passes read it with LDS instead of an L1 LDG per step, which ptxas
  // schedules next to its use instead of hoisting it beside the y loads
  extern __shared__ double2 gsu[];
  // allow_factor & 4: fit_grid_ring_kernel took the f3-periodic grouped grid
  if (KIND == DOOLY_KIND_ATTN && (allow_factor & 4) && gf->ok && gf->grp4 && gf->f3p128 &&
      n_pts % kRingPts == 0)
    return;

  __shared__ double sW[NC][NC];
  __shared__ double sinv[P];
  __shared__ uint32_t slo[P], shi[P];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int t = tid; t < NC * NC; t += blockDim.x) sW[t / NC][t % NC] = gf->W[t / NC][t % NC];
  if (tid < P) {
    sinv[tid] = gf->inv[tid];
    slo[tid] = gf->lo[tid];
    shi[tid] = gf->hi[tid];
  }
  const bool ok = gf->ok != 0;
  const bool factored = KIND == DOOLY_KIND_ATTN && (allow_factor & 3) && gf->grp4 != 0;
  const bool f3reg = factored && gf->f3p128 != 0;
  __syncthreads();
  const bool su = factored && su_groups > 0;
  if (su) {
    const double2* g2 = reinterpret_cast<const double2*>(fpl + 3 * n_pts);
    for (int g = tid; g < su_groups; g += blockDim.x) gsu[g] = g2[g];
    __syncthreads();
  }
  double inv[P], nb[P];
#pragma unroll
  for (int k = 0; k < P; ++k) inv[k] = sinv[k], nb[k] = -4503599627370496.0 * sinv[k];
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + tid) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int n = (int)n_pts;  // n_pts % 4 == 0, n_pts < 2^31 (launcher)
  const double4 f3l = f3reg ? g_ld_f(fpl + 2 * n + 4 * lane) : make_double4(0.0, 0.0, 0.0, 0.0);
  for (int64_t s = warp; s < n_sig; s += n_warps) {
    if (!ok) {
      if (lane == 0) write_unfitted_grid<KIND>(pe, gf, table, s, fit_err, status);
      continue;
    }
    const double* ys = y + s * n_pts;
    // ---- pass 1: b = M^T y, 4 consecutive points per lane per step
    double acc[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) acc[k] = 0.0;
    auto pass1_step = [&](const double4& yv, const double4* fv) {
      const double yy[4] = {yv.x, yv.y, yv.z, yv.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        double f[P];
#pragma unroll
        for (int k = 0; k < P; ++k)
          f[k] = j == 0 ? fv[k].x : j == 1 ? fv[k].y : j == 2 ? fv[k].z : fv[k].w;
        if constexpr (KIND == DOOLY_KIND_AFFINE) {
          acc[0] += yy[j];
          acc[1] = fma(yy[j], f[0], acc[1]);
        } else {
          const double y1 = yy[j] * f[0], y2 = yy[j] * f[1], y3 = yy[j] * f[2];
          acc[0] += yy[j];
          acc[1] += y1;
          acc[2] += y2;
          acc[3] += y3;
          acc[4] = fma(y1, f[0], acc[4]);
          acc[5] = fma(y2, f[1], acc[5]);
          acc[6] = fma(y3, f[2], acc[6]);
          acc[7] = fma(y1, f[1], acc[7]);
          acc[8] = fma(y1, f[2], acc[8]);
          acc[9] = fma(y2, f[2], acc[9]);
        }
      }
    };
    double c[NC];
    double err = 0.0;
    auto pass2_step = [&](const double4& yv, const double4* fv) {
      const double yy[4] = {yv.x, yv.y, yv.z, yv.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        double f[P];
#pragma unroll
        for (int k = 0; k < P; ++k)
          f[k] = j == 0 ? fv[k].x : j == 1 ? fv[k].y : j == 2 ? fv[k].z : fv[k].w;
        const double pr = fmax(grid_horner<KIND>(c, f), DOOLY_CLAMP_FLOOR);
        err = fma(fabs(pr - yy[j]), g_rcp1(yy[j]), err);
      }
    };
    // One pass over the row: 4 consecutive points per lane per step, y from
    // HBM/L2 and the scaled features f from the L1-resident planes.  YS steps
    // of y (8 x 32 B per lane) are issued before any of their math, f is
    // loaded per step (an L1 hit); the tail runs two steps, then one.
    // Measured (0.5M signatures x 4096 points): YS = 2 -> 8 took attention
    // from 5.75 to 5.11 ms and affine from 2.92 to 2.85 ms; 12 and 16 were slower.
    auto ldf = [&](int p, double4* fv) {
#pragma unroll
      for (int k = 0; k < P; ++k) fv[k] = g_ld_f(fpl + k * n + p);
    };
    auto sweep = [&](bool keep, auto&& step) {
      int p = 4 * lane;
      constexpr int YS = FG_WARP_YS;
      for (; p + 128 * (YS - 1) < n; p += 128 * YS) {
        double4 yv[YS];
#pragma unroll
        for (int t = 0; t < YS; ++t) yv[t] = g_ld_y(ys + p + 128 * t, keep);
#pragma unroll
        for (int t = 0; t < YS; ++t) {
          double4 fv[P];
          ldf(p + 128 * t, fv);
          step(yv[t], fv);
        }
      }
      for (; p + 128 < n; p += 256) {
        const double4 ya = g_ld_y(ys + p, keep), yb = g_ld_y(ys + p + 128, keep);
        double4 fa[P], fb[P];
        ldf(p, fa);
        ldf(p + 128, fb);
        step(ya, fa);
        step(yb, fb);
      }
      if (p < n) {
        const double4 ya = g_ld_y(ys + p, keep);
        double4 fa[P];
        ldf(p, fa);
        step(ya, fa);
      }
    };
    if (factored) {
      // Pass 1 on a grid whose aligned 4-point groups share f1 and f2 (prep's
      // grp4): per group the kv sums s0 = sum y, s1 = sum y f3, s2 = sum y f3^2
      // (4 FP64 per point), then the 10 moments as s_c times the group's f1^a f2^b
      // (13 FP64 per group) — 7.25 FP64 per point instead of 13, and one
      // feature plane read per step instead of three.  Pass 2 likewise folds
      // the f1/f2 terms per group: 8.75 FP64 per point instead of 14.
      // f3 source as a compile-time choice: the lane's register quad (f3reg)
      // or an L1 load — a runtime select would copy the quad into the load's
      // destination registers before every predicated load (8 moves a step)
      auto pass1 = [&](auto f3of) {
        auto fstep = [&](const double4& yv, int pp) {
          const double2 u = __ldg(reinterpret_cast<const double2*>(fpl + 3 * n) + (pp >> 2));
          grid_g1_step(yv, f3of(pp), u.x, u.y, acc);
        };
        int p = 4 * lane;
        constexpr int YS = FG_WARP_YS;
        for (; p + 128 * (YS - 1) < n; p += 128 * YS) {
          double4 yv[YS];
#pragma unroll
          for (int t = 0; t < YS; ++t) yv[t] = g_ld_y(ys + p + 128 * t, true);
#pragma unroll
          for (int t = 0; t < YS; ++t) fstep(yv[t], p + 128 * t);
        }
        for (; p < n; p += 128) fstep(g_ld_y(ys + p, true), p);
      };
      if (f3reg && (allow_factor & 3) >= 2) {
        // f3 fixed per lane position: per-position sums, f3 folded in once
        auto run_r1 = [&](auto uof) {
          GridR1 r1;
#pragma unroll
          for (int j = 0; j < 4; ++j) r1.T[j] = r1.U1[j] = r1.U2[j] = 0.0;
          r1.Q[0] = r1.Q[1] = r1.Q[2] = 0.0;
          auto rstep = [&](const double4& yv, int pp) {
            const double2 u = uof(pp);
            grid_r1_step(yv, u.x, u.y, r1);
          };
          int p = 4 * lane;
          constexpr int YS = FG_WARP_YS;
          for (; p + 128 * (YS - 1) < n; p += 128 * YS) {
            double4 yv[YS];
#pragma unroll
            for (int t = 0; t < YS; ++t) yv[t] = g_ld_y(ys + p + 128 * t, true);
#pragma unroll
            for (int t = 0; t < YS; ++t) rstep(yv[t], p + 128 * t);
          }
          for (; p < n; p += 128) rstep(g_ld_y(ys + p, true), p);
          grid_r1_fold(r1, f3l, acc);
        };
        if (su)
          run_r1([&](int pp) { return gsu[pp >> 2]; });
        else
          run_r1([&](int pp) {
            return __ldg(reinterpret_cast<const double2*>(fpl + 3 * n) + (pp >> 2));
          });
      } else if (f3reg) {
        pass1([&](int) { return f3l; });
      } else {
        pass1([&](int pp) { return g_ld_f(fpl + 2 * n + pp); });
      }
    } else {
      sweep(true, pass1_step);
    }
#pragma unroll
    for (int k = 0; k < NC; ++k) acc[k] = g_warp_sum(acc[k]);
    // ---- c = W b: lane j < NC forms coefficient j, then broadcast
    double cj = 0.0;
    if (lane < NC) {
#pragma unroll
      for (int i = 0; i < NC; ++i) cj = fma(sW[lane][i], acc[i], cj);
    }
#pragma unroll
    for (int k = 0; k < NC; ++k) c[k] = __shfl_sync(0xFFFFFFFFu, cj, k);
    // ---- pass 2: training MAPE, the row re-read from L2
    if (factored) {
      // per group: p = A + f3 (B + c6 f3) with A, B the group's f1/f2 terms
      auto pass2 = [&](auto f3of, auto uof) {
        auto fstep2 = [&](const double4& yv, int pp) {
          const double2 u = uof(pp);
          grid_g2_step(yv, f3of(pp), u.x, u.y, c, err);
        };
        int p = 4 * lane;
        constexpr int YS = FG_WARP_YS;
        for (; p + 128 * (YS - 1) < n; p += 128 * YS) {
          double4 yv[YS];
#pragma unroll
          for (int t = 0; t < YS; ++t) yv[t] = g_ld_y(ys + p + 128 * t, false);
#pragma unroll
          for (int t = 0; t < YS; ++t) fstep2(yv[t], p + 128 * t);
        }
        for (; p < n; p += 128) fstep2(g_ld_y(ys + p, false), p);
      };
      auto ug = [&](int pp) {
        return __ldg(reinterpret_cast<const double2*>(fpl + 3 * n) + (pp >> 2));
      };
      if (f3reg && su)
        pass2([&](int) { return f3l; }, [&](int pp) { return gsu[pp >> 2]; });
      else if (f3reg)
        pass2([&](int) { return f3l; }, ug);
      else
        pass2([&](int pp) { return g_ld_f(fpl + 2 * n + pp); }, ug);
    } else {
      sweep(false, pass2_step);
    }
    err = g_warp_sum(err);
    if (lane == 0)
      emit_row<KIND>(pe, gf, table, fit_err, status, s, make_row<KIND>(c, sinv, slo, shi),
                     err / (double)n_pts, DOOLY_FIT_OK);
  }
}

// Per-step arithmetic of the two passes (4 consecutive points per lane), the
// same operations in the same order as fit_grid_warp_kernel's lambdas.
template <int KIND>
__device__ __forceinline__ void grid_p1_step(const double4& yv, const double4* fv, double* acc) {
  constexpr int P = KIND == DOOLY_KIND_AFFINE ? 1 : 3;
  const double yy[4] = {yv.x, yv.y, yv.z, yv.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    double f[P];
#pragma unroll
    for (int k = 0; k < P; ++k) f[k] = j == 0 ? fv[k].x : j == 1 ? fv[k].y : j == 2 ? fv[k].z : fv[k].w;
    if constexpr (KIND == DOOLY_KIND_AFFINE) {
      acc[0] += yy[j];
      acc[1] = fma(yy[j], f[0], acc[1]);
    } else {
      const double y1 = yy[j] * f[0], y2 = yy[j] * f[1], y3 = yy[j] * f[2];
      acc[0] += yy[j];
      acc[1] += y1;
      acc[2] += y2;
      acc[3] += y3;
      acc[4] = fma(y1, f[0], acc[4]);
      acc[5] = fma(y2, f[1], acc[5]);
      acc[6] = fma(y3, f[2], acc[6]);
      acc[7] = fma(y1, f[1], acc[7]);
      acc[8] = fma(y1, f[2], acc[8]);
      acc[9] = fma(y2, f[2], acc[9]);
    }
  }
}

template <int KIND>
__device__ __forceinline__ void grid_p2_step(const double4& yv, const double4* fv, const double* c,
                                             double& err) {
  constexpr int P = KIND == DOOLY_KIND_AFFINE ? 1 : 3;
  const double yy[4] = {yv.x, yv.y, yv.z, yv.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    double f[P];
#pragma unroll
    for (int k = 0; k < P; ++k) f[k] = j == 0 ? fv[k].x : j == 1 ? fv[k].y : j == 2 ? fv[k].z : fv[k].w;
    const double pr = fmax(grid_horner<KIND>(c, f), DOOLY_CLAMP_FLOOR);
    err = fma(fabs(pr - yy[j]), g_rcp1(yy[j]), err);
  }
}

// Register double-buffered sweep (n % (128 * YS) == 0): the loads of batch
// k + 1 (YS steps of y per lane) are in flight while batch k is evaluated, so
// a lane always has between YS and 2 YS steps outstanding.
template <int KIND, int YS, bool P1, bool GROUPED = false>
__device__ __forceinline__ void grid_sweep_db(const double* __restrict__ fpl, int n, int lane,
                                              const double* yr, const double* c, double* acc,
                                              double& err) {
  constexpr int P = KIND == DOOLY_KIND_AFFINE ? 1 : 3;
  constexpr int S = 128 * YS;
  double4 va[YS], vb[YS];
  auto load = [&](double4* v, int p) {
#pragma unroll
    for (int t = 0; t < YS; ++t) v[t] = g_ld_y(yr + p + 128 * t, P1);
  };
  auto eval = [&](const double4* v, int p) {
#pragma unroll
    for (int t = 0; t < YS; ++t) {
      const int q = p + 128 * t;
      if constexpr (GROUPED) {
        const double4 f3 = g_ld_f(fpl + 2 * n + q);
        const double2 u = __ldg(reinterpret_cast<const double2*>(fpl + 3 * n) + (q >> 2));
        const double u1 = u.x, u2 = u.y;
        if (P1)
          grid_g1_step(v[t], f3, u1, u2, acc);
        else
          grid_g2_step(v[t], f3, u1, u2, c, err);
      } else {
        double4 fv[P];
#pragma unroll
        for (int k = 0; k < P; ++k) fv[k] = g_ld_f(fpl + k * n + q);
        if (P1)
          grid_p1_step<KIND>(v[t], fv, acc);
        else
          grid_p2_step<KIND>(v[t], fv, c, err);
      }
    }
  };
  int p = 4 * lane;
  load(va, p);
  for (; p + S < n; p += 2 * S) {
    load(vb, p + S);
    eval(va, p);
    if (p + 2 * S < n) load(va, p + 2 * S);
    eval(vb, p + S);
  }
  if (p < n) eval(va, p);
}

template <int KIND, int YS>
__global__ void __launch_bounds__(256, 2) fit_grid_db_kernel(
    const double* __restrict__ fpl, int64_t n_pts, const double* __restrict__ y, int64_t n_sig,
    const GridFactor* __restrict__ gf, void* __restrict__ table, double* __restrict__ fit_err,
    uint8_t* __restrict__ status, const GridOut pe, int allow_factor) {
  using T = GridTraits<KIND>;
  constexpr int P = T::P, NC = T::NC;
  __shared__ double sW[NC][NC];
  __shared__ double sinv[P];
  __shared__ uint32_t slo[P], shi[P];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int t = tid; t < NC * NC; t += blockDim.x) sW[t / NC][t % NC] = gf->W[t / NC][t % NC];
  if (tid < P) {
    sinv[tid] = gf->inv[tid];
    slo[tid] = gf->lo[tid];
    shi[tid] = gf->hi[tid];
  }
  const bool ok = gf->ok != 0;
  __syncthreads();
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + tid) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int n = (int)n_pts;  // n_pts % (128 * YS) == 0 (launcher)
  for (int64_t s = warp; s < n_sig; s += n_warps) {
    if (!ok) {
      if (lane == 0) write_unfitted_grid<KIND>(pe, gf, table, s, fit_err, status);
      continue;
    }
    const double* ys = y + s * n_pts;
    double acc[NC], c[NC];
    double err = 0.0;
#pragma unroll
    for (int k = 0; k < NC; ++k) acc[k] = 0.0;
    if (KIND == DOOLY_KIND_ATTN && allow_factor && gf->grp4 != 0)
      grid_sweep_db<KIND, YS, true, KIND == DOOLY_KIND_ATTN>(fpl, n, lane, ys, c, acc, err);
    else
      grid_sweep_db<KIND, YS, true>(fpl, n, lane, ys, c, acc, err);
#pragma unroll
    for (int k = 0; k < NC; ++k) acc[k] = g_warp_sum(acc[k]);
    double cj = 0.0;
    if (lane < NC) {
#pragma unroll
      for (int i = 0; i < NC; ++i) cj = fma(sW[lane][i], acc[i], cj);
    }
#pragma unroll
    for (int k = 0; k < NC; ++k) c[k] = __shfl_sync(0xFFFFFFFFu, cj, k);
    if (KIND == DOOLY_KIND_ATTN && allow_factor && gf->grp4 != 0)
      grid_sweep_db<KIND, YS, false, KIND == DOOLY_KIND_ATTN>(fpl, n, lane, ys, c, acc, err);
    else
      grid_sweep_db<KIND, YS, false>(fpl, n, lane, ys, c, acc, err);
    err = g_warp_sum(err);
    if (lane == 0)
      emit_row<KIND>(pe, gf, table, fit_err, status, s, make_row<KIND>(c, sinv, slo, shi),
                     err / (double)n_pts, DOOLY_FIT_OK);
  }
}

// ---- warp-specialised attention grid fit (opt-in, DOOLY_FIT_GRID_KERNEL=ws /
// ws8 / ws3; measured slower than fit_grid_warp_kernel, see the launcher and
// profiles/r2_fit_grid_ws.md).  One persistent CTA per SM: warp 0 is the
// PRODUCER — lane 0 bulk-copies (1-D TMA, cp.async.bulk + mbarrier
// complete_tx) whole y rows of the CTA's signatures into an S-stage shared
// memory ring — and the other WSG x WSW warps are CONSUMERS in WSG groups, group
// g fitting the CTA's signatures k = g, g + WSG, ...  A group fits one
// signature with all its threads: each thread keeps the scaled features of
// ITS points in registers for the whole launch (the grid is shared by every
// signature), reads the row's y from shared memory in both passes (pass 2
// re-reads smem instead of L2), and the group reduces b and the MAPE through
// shared memory behind a named barrier; thread 0 emits the row and releases
// the stage to the producer.  y crosses HBM once, always with a ring of rows
// in flight, and no consumer ever waits on a global load.  The arithmetic is
// exactly fit_grid_warp_kernel's (grouped passes when the grid is grp4,
// per-point passes otherwise), only the summation order differs.
constexpr size_t kWsRing = 160 * 1024;               // y ring bytes

template <int kWsGroups, int kWsWarps>
__global__ void __launch_bounds__(32 + kWsGroups * kWsWarps * 32, 1) fit_grid_ws_kernel(
    const double* __restrict__ fpl, int64_t n_pts, const double* __restrict__ y, int64_t n_sig,
    const GridFactor* __restrict__ gf, void* __restrict__ table, double* __restrict__ fit_err,
    uint8_t* __restrict__ status, const GridOut pe, int allow_factor, int n_stage) {
  constexpr int KIND = DOOLY_KIND_ATTN, NC = 10;
  constexpr int kWsGT = kWsWarps * 32;                 // threads per group
  constexpr int kWsMaxG = 32 / kWsWarps;               // 4-point groups per thread (n_pts <= 4096)
  extern __shared__ __align__(128) unsigned char wsdyn[];
  double* ring = reinterpret_cast<double*>(wsdyn);
  __shared__ __align__(8) uint64_t full[8], empty[8];
  __shared__ double sW[NC][NC];
  __shared__ double part[kWsGroups][kWsWarps][NC + 1];
  __shared__ double scoef[kWsGroups][NC];
  __shared__ double sinv[3];
  __shared__ uint32_t slo[3], shi[3];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int t = tid; t < NC * NC; t += blockDim.x) sW[t / NC][t % NC] = gf->W[t / NC][t % NC];
  if (tid < 3) {
    sinv[tid] = gf->inv[tid];
    slo[tid] = gf->lo[tid];
    shi[tid] = gf->hi[tid];
  }
  if (tid == 0) {
    for (int i = 0; i < n_stage; ++i) {
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(g_smem(&full[i])));
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(g_smem(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const bool ok = gf->ok != 0;
  const bool grouped = allow_factor && gf->grp4 != 0;
  const int n = (int)n_pts;
  const int64_t n_mine = n_sig > blockIdx.x ? (n_sig - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const uint32_t row_bytes = (uint32_t)n * 8u;

  if (wid == 0) {  // ---------------- producer
    if (lane == 0 && ok) {
      for (int64_t k = 0; k < n_mine; ++k) {
        const int st = (int)(k % n_stage);
        if (k >= n_stage) g_wait(&empty[st], (uint32_t)(((k / n_stage) - 1) & 1));
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(g_smem(&full[st])),
                     "r"(row_bytes)
                     : "memory");
        const int64_t s = blockIdx.x + k * gridDim.x;
        g_bulk(ring + (size_t)st * n, y + s * n_pts, row_bytes, &full[st]);
      }
    }
    return;
  }
  // ---------------- consumers
  const int g = (wid - 1) / kWsWarps, gw = (wid - 1) % kWsWarps, gt = tid - 32 - g * kWsGT;
  const int ngr = n / (4 * kWsGT);  // 4-point groups per thread (launcher: 1..kWsMaxG)
  // this thread's points: groups q = gt + kWsGT * j, points 4q .. 4q + 3
  // (f3 per point and the group's (u1, u2) in registers; the per-point passes
  // of a non-grp4 grid read f1 / f2 from the L1-resident planes)
  double4 f3r[kWsMaxG];
  double2 ur[kWsMaxG];
#pragma unroll
  for (int j = 0; j < kWsMaxG; ++j) {
    if (j < ngr) {
      const int q = gt + kWsGT * j;
      f3r[j] = g_ld_f(fpl + 2 * n + 4 * q);
      ur[j] = grouped ? __ldg(reinterpret_cast<const double2*>(fpl + 3 * n) + q)
                      : make_double2(0.0, 0.0);
    }
  }
  const int bar_id = 1 + g;
  auto group_sync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(kWsGT) : "memory"); };
  for (int64_t k = g; k < n_mine; k += kWsGroups) {
    const int64_t s = blockIdx.x + k * gridDim.x;
    if (!ok) {
      if (gt == 0) write_unfitted_grid<KIND>(pe, gf, table, s, fit_err, status);
      continue;
    }
    const int st = (int)(k % n_stage);
    g_wait(&full[st], (uint32_t)((k / n_stage) & 1));
    const double* yr = ring + (size_t)st * n;
    double acc[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) acc[i] = 0.0;
#pragma unroll
    for (int j = 0; j < kWsMaxG; ++j) {
      if (j < ngr) {
        const double4 yv = *reinterpret_cast<const double4*>(yr + 4 * (gt + kWsGT * j));
        if (grouped) {
          grid_g1_step(yv, f3r[j], ur[j].x, ur[j].y, acc);
        } else {
          const int q = gt + kWsGT * j;
          const double4 fv[3] = {g_ld_f(fpl + 4 * q), g_ld_f(fpl + n + 4 * q), f3r[j]};
          grid_p1_step<KIND>(yv, fv, acc);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < NC; ++i) acc[i] = g_warp_sum(acc[i]);
    if (lane == 0)
#pragma unroll
      for (int i = 0; i < NC; ++i) part[g][gw][i] = acc[i];
    group_sync();
    if (gt < NC) {  // c = W b: thread j forms coefficient j
      double b[NC];
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        double v = 0.0;
#pragma unroll
        for (int w = 0; w < kWsWarps; ++w) v += part[g][w][i];
        b[i] = v;
      }
      double cj = 0.0;
#pragma unroll
      for (int i = 0; i < NC; ++i) cj = fma(sW[gt][i], b[i], cj);
      scoef[g][gt] = cj;
    }
    group_sync();
    double c[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) c[i] = scoef[g][i];
    double err = 0.0;
#pragma unroll
    for (int j = 0; j < kWsMaxG; ++j) {
      if (j < ngr) {
        const double4 yv = *reinterpret_cast<const double4*>(yr + 4 * (gt + kWsGT * j));
        if (grouped) {
          grid_g2_step(yv, f3r[j], ur[j].x, ur[j].y, c, err);
        } else {
          const int q = gt + kWsGT * j;
          const double4 fv[3] = {g_ld_f(fpl + 4 * q), g_ld_f(fpl + n + 4 * q), f3r[j]};
          grid_p2_step<KIND>(yv, fv, c, err);
        }
      }
    }
    err = g_warp_sum(err);
    if (lane == 0) part[g][gw][NC] = err;
    group_sync();  // every read of the stage and of scoef is done
    if (gt == 0) {
      asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(g_smem(&empty[st])) : "memory");
      double e = 0.0;
#pragma unroll
      for (int w = 0; w < kWsWarps; ++w) e += part[g][w][NC];
      emit_row<KIND>(pe, gf, table, fit_err, status, s, make_row<KIND>(c, sinv, slo, shi),
                     e / (double)n_pts, DOOLY_FIT_OK);
    }
  }
}

template <int KIND>
static cudaError_t launch_grid_kind(const uint32_t* x, int64_t n_pts, const double* y, int64_t n_sig,
                                    void* table, double* fit_err, uint8_t* status,
                                    const GridOut& pe, void* ws, cudaStream_t stream,
                                    int n_sm, int64_t* launches) {
  GridFactor* gf = static_cast<GridFactor*>(ws);
  double* fpl = reinterpret_cast<double*>(static_cast<char*>(ws) + grid_factor_bytes());
  fit_grid_prep_kernel<KIND><<<1, kGT, 0, stream>>>(x, n_pts, gf, fpl, pe.packed, pe.row0 + n_sig);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  *launches += 1;
  if (n_sig == 0) return cudaSuccess;
  // "db" (default for affine) | "warp" (default for attention) | "ws"/"ws8"/"ws3" | "stage" | "plain"
  const char* which = getenv("DOOLY_FIT_GRID_KERNEL");
  // "0": per-point attention passes; "1": grouped passes without the
  // per-position pass 1 (grid_r1_step) on f3-periodic grids
  const char* fac = getenv("DOOLY_FIT_GRID_FACTOR");
  const int allow_factor = fac == nullptr ? 2 : fac[0] == '0' ? 0 : fac[0] == '1' ? 1 : 2;
  const bool aligned = n_pts < (1ll << 30) && (uintptr_t)y % 32 == 0 && (uintptr_t)ws % 32 == 0;
  // warps in flight x row bytes must stay well inside L2 so pass 2 re-reads hit
  const int warps_per_sm =
      getenv("DOOLY_FIT_GRID_WARPS") ? atoi(getenv("DOOLY_FIT_GRID_WARPS")) : 16;
  const int64_t warp_blocks =
      std::min<int64_t>((int64_t)n_sm * (warps_per_sm > 8 ? warps_per_sm / 8 : 1), (n_sig + 7) / 8);
  // Double-buffered warp kernel: measured 2.70 vs 2.78 ms (affine) and 5.39 vs
  // 5.12 ms (attention) per 0.5M signatures x 4096 points against the warp
  // kernel, so it is the affine default only.
  const bool want_db = which != nullptr ? strcmp(which, "db") == 0 : KIND == DOOLY_KIND_AFFINE;
  if (want_db && aligned && n_pts % 256 == 0) {
    auto kern = n_pts % 512 == 0 ? fit_grid_db_kernel<KIND, 4> : fit_grid_db_kernel<KIND, 2>;
    kern<<<(unsigned)warp_blocks, 256, 0, stream>>>(fpl, n_pts, y, n_sig, gf, table, fit_err,
                                                    status, pe, allow_factor & 3);
    *launches += 1;
    return cudaGetLastError();
  }
  // warp-specialised TMA ring (attention default): whole rows <= 32 KB,
  // n_pts a multiple of 512 (4-point groups spread evenly over a group's threads)
  // opt-in (measured 6.85 ms vs the warp kernel's 3.69 ms per 0.5M x 4096
  // attention points: two or three consumer warps per SMSP cannot hide the
  // FP64 dependency chains; profiles/r2_fit_grid_ws.md)
  const bool want_ws = which != nullptr && strncmp(which, "ws", 2) == 0;
  // variants: "ws" 2 groups x 4 warps, "ws8" 2 x 8, "ws3" 3 x 4
  const int wsw = which != nullptr && strcmp(which, "ws8") == 0 ? 8 : 4;
  const int wsg = which != nullptr && strcmp(which, "ws3") == 0 ? 3 : 2;
  if (KIND == DOOLY_KIND_ATTN && want_ws && aligned && n_pts % (4 * 32 * wsw) == 0 &&
      n_pts / (4 * 32 * wsw) <= 32 / wsw) {
    const int n_stage = (int)std::min<int64_t>(8, kWsRing / (n_pts * 8));
    const size_t smem = (size_t)n_stage * n_pts * 8;
    auto kern = wsw == 8 ? fit_grid_ws_kernel<2, 8>
              : wsg == 3 ? fit_grid_ws_kernel<3, 4> : fit_grid_ws_kernel<2, 4>;
    cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem);
    if (e2 != cudaSuccess) return e2;
    const int64_t blocks = std::min<int64_t>(n_sm, std::max<int64_t>(1, n_sig));
    kern<<<(unsigned)blocks, 32 + wsg * wsw * 32, smem, stream>>>(
        fpl, n_pts, y, n_sig, gf, table, fit_err, status, pe, allow_factor & 3, n_stage);
    *launches += 1;
    return cudaGetLastError();
  }
  // per-warp bulk-copy ring for f3-periodic grouped grids (the grid's
  // properties are known on the device only: the ring kernel returns at once
  // on other grids and the warp kernel, launched after it, skips the ring's case)
  const bool want_ring = which != nullptr && strncmp(which, "ring", 4) == 0;
  int ring_flag = 0;
  if (KIND == DOOLY_KIND_ATTN && want_ring && (allow_factor & 3) == 2 && aligned &&
      n_pts % kRingPts == 0) {
    // "ring": 3 x 4 KB stages, 2 CTAs/SM; "ring6": 6 x 2 KB; "ring2": 2 x 4 KB, 3 CTAs/SM
    const int v = strcmp(which, "ring6") == 0 ? 1 : strcmp(which, "ring2") == 0 ? 2 : 0;
    auto kern = v == 1 ? fit_grid_ring_kernel<6, 2048, 2>
              : v == 2 ? fit_grid_ring_kernel<2, 4096, 3> : fit_grid_ring_kernel<3, 4096, 2>;
    const int per_sm = v == 2 ? 3 : 2;
    const size_t smem = (size_t)8 * (v == 1 ? 6 * 2048 : v == 2 ? 2 * 4096 : 3 * 4096);
    cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem);
    if (e2 != cudaSuccess) return e2;
    const int64_t blocks = std::min<int64_t>((int64_t)n_sm * per_sm, (n_sig + 7) / 8);
    kern<<<(unsigned)blocks, 256, smem, stream>>>(fpl, n_pts, y, n_sig, gf, table, fit_err,
                                                  status, pe);
    *launches += 1;
    e2 = cudaGetLastError();
    if (e2 != cudaSuccess) return e2;
    ring_flag = 4;
  }
  const bool want_warp = which == nullptr || which[0] == 'w' || which[0] == 'd' || want_ring;
  if (want_warp && n_pts % 4 == 0 && aligned) {
    // attention: the group plane in shared memory when it is small (C5: 16 KB)
    const int su_groups = KIND == DOOLY_KIND_ATTN && getenv("DOOLY_FIT_GRID_SU0") == nullptr &&
                                  n_pts <= 8192 ? (int)(n_pts / 4) : 0;
    fit_grid_warp_kernel<KIND><<<(unsigned)warp_blocks, 256, (size_t)su_groups * 16, stream>>>(
        fpl, n_pts, y, n_sig, gf, table, fit_err, status, pe, allow_factor | ring_flag, su_groups);
    *launches += 1;
    return cudaGetLastError();
  }
  const size_t stage = (size_t)GridTraits<KIND>::RS * n_pts * 8;
  const bool no_stage = which != nullptr && strcmp(which, "plain") == 0;
  if (!no_stage && stage <= kGridStageMax && n_pts % 4 == 0 && (uintptr_t)y % 16 == 0) {
    auto kern = fit_grid_stage_kernel<KIND>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGridStageMax);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kGT, stage);
    const int64_t groups = (n_sig + GridTraits<KIND>::RS - 1) / GridTraits<KIND>::RS;
    int64_t blocks = (int64_t)n_sm * (per_sm > 0 ? per_sm : 1);
    if (blocks > groups) blocks = groups;
    kern<<<(unsigned)blocks, kGT, stage, stream>>>(x, n_pts, y, n_sig, gf, table, fit_err,
                                                   status, pe);
    *launches += 1;
    return cudaGetLastError();
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fit_grid_kernel<KIND>, kGT, 0);
  const int64_t groups = (n_sig + GridTraits<KIND>::R - 1) / GridTraits<KIND>::R;
  int64_t blocks = (int64_t)n_sm * (per_sm > 0 ? per_sm : 1);
  if (blocks > groups) blocks = groups;
  fit_grid_kernel<KIND><<<(unsigned)blocks, kGT, 0, stream>>>(x, n_pts, y, n_sig, gf, table,
                                                              fit_err, status, pe);
  *launches += 1;
  return cudaGetLastError();
}

// Workspace: the GridFactor, then the scaled feature planes f_k(p) = RN(x_k(p) * inv_k)
// (P x n_pts f64) that the warp kernel reads instead of converting x per point,
// then (attention) the (f1, f2) plane of the aligned 4-point groups.
size_t fit_grid_workspace_size(int kind, int64_t n_pts) {
  const int P = kind == DOOLY_KIND_AFFINE ? 1 : 3;
  const size_t n = (size_t)(n_pts > 0 ? n_pts : 0);
  // attention: + the (f1, f2) group plane of the grouped passes
  return grid_factor_bytes() + (size_t)P * n * 8 + (kind == DOOLY_KIND_AFFINE ? 0 : (n / 4) * 16);
}

cudaError_t launch_fit_grid(int kind, const uint32_t* x, int64_t n_pts, const double* y,
                            int64_t n_sig, void* table, double* fit_err, uint8_t* status,
                            const dooly_grid_peers* peers, void* ws, cudaStream_t stream,
                            int n_sm, int64_t* launches, void* packed) {
  GridOut pe{};
  if (peers) static_cast<dooly_grid_peers&>(pe) = *peers;
  pe.packed = static_cast<uint8_t*>(packed);
  if (kind == DOOLY_KIND_AFFINE)
    return launch_grid_kind<DOOLY_KIND_AFFINE>(x, n_pts, y, n_sig, table, fit_err, status, pe, ws,
                                               stream, n_sm, launches);
  return launch_grid_kind<DOOLY_KIND_ATTN>(x, n_pts, y, n_sig, table, fit_err, status, pe, ws,
                                           stream, n_sm, launches);
}

}  // namespace dooly
