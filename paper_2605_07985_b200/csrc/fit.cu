// K2 — batched per-signature least-squares fit (replaces fit).
//
// Data path (B200): a persistent kernel with two 128-thread CTAs per SM.  In
// each CTA thread 0 streams whole signatures (feature planes + latencies) from
// HBM into a ring of shared-memory stages with the bulk-copy (1-D TMA) engine
// (`cp.async.bulk` + mbarrier complete_tx), so both passes over a signature
// read shared memory and every point is fetched from HBM exactly once.  The
// two co-resident CTAs interleave: while one is in its short serial phase
// (reduce + solve) or waiting for its next stage, the other keeps the FP64
// pipes busy.  Signatures larger than a stage (or unaligned inputs) fall back
// to a direct global-memory path with the same arithmetic.
//
// Per signature:
//   pass 1  raw power moments sum x^a y^b z^c (a+b+c <= 4: 34 non-trivial for
//           attention, 2 for affine) and X^T y for the design monomials, plus
//           the training box.  All terms are non-negative, so the raw sums are
//           well conditioned; the scaled Gram G[i][j] = M[e_i+e_j] * prod inv^e
//           is formed once per signature.  Degree-4 monomials are leaves and go
//           straight into their accumulator with one FMA (63 FP64 instructions
//           per attention point instead of ~130 for a direct 10x10 Gram).
//           u32 -> f64 conversion uses the exact 2^52 bias trick (one DADD on
//           the FP64 pipe instead of the quarter-rate I2F).
//   reduce  warp shuffles -> shared memory -> warp 0.
//   solve   warp 0 factors G with a right-looking Cholesky, one lane per row,
//           reciprocal-multiply instead of FP64 division; columns whose pivot
//           falls to <= DROP_TOL x their diagonal are dropped (rank-deficient
//           designs), then forward/back substitution by shuffles.
//   pass 2  training MAPE (fit_error) of the clamped predictor (FMA form; the
//           bit-exact no-FMA form is only needed where predictions are
//           returned, see common.cuh).
// FP64 throughout; no tensor cores (B200's FP64 tensor peak equals the FP64
// vector peak and lower precisions cannot meet the 1e-9 contract).
#include <stdlib.h>

#include "attn_moments.cuh"
#include "common.cuh"

namespace dooly {

constexpr double DROP_TOL = 1e-9;
constexpr int FIT_CAP = 4096;  // points per shared-memory stage
constexpr int FIT_CTAS_PER_SM = 2;

template <int KIND>
struct FitTraits;

template <>
struct FitTraits<DOOLY_KIND_AFFINE> {
  static constexpr int P = 1;      // features
  static constexpr int NCOL = 2;   // design columns [1, f]
  static constexpr int NMOM = 3;   // 1, x, x^2
  static constexpr int NEED = 4;   // max(4, NCOL + 1)   (App. A.8)
  static constexpr int STAGES = 1;  // 4 CTAs/SM x 1 stage beat 2x2 and 1x3 (profiles/)
  static constexpr int THREADS = 128;
  static constexpr int SETS = 2;  // independent accumulator sets (breaks DADD chains)
  __device__ static __forceinline__ void accumulate(const double* v, double y, double* acc) {
    acc[0] += v[0];
    acc[1] = fma(v[0], v[0], acc[1]);
    acc[2] += y;
    acc[3] = fma(y, v[0], acc[3]);
  }
};

template <>
struct FitTraits<DOOLY_KIND_ATTN> {
  static constexpr int P = 3;
  static constexpr int NCOL = 10;
  static constexpr int NMOM = 35;
  static constexpr int NEED = 11;
  static constexpr int STAGES = 1;
  static constexpr int THREADS = 128;
  static constexpr int SETS = 1;  // 44 independent accumulators already give the ILP
  __device__ static __forceinline__ void accumulate(const double* v, double y, double* acc) {
    attn_accumulate(v[0], v[1], v[2], y, acc);
  }
};

// Stage layout in shared memory: y[FIT_CAP + 2] f64, then P planes of
// x[FIT_CAP + 4] u32 (the +2/+4 hold the head misalignment of the window).
template <int KIND>
struct Stage {
  static constexpr int P = FitTraits<KIND>::P;
  static constexpr int Y_LEN = FIT_CAP + 2;
  static constexpr int X_LEN = FIT_CAP + 4;
  static constexpr size_t BYTES = (size_t)Y_LEN * 8 + (size_t)P * X_LEN * 4;
  static constexpr size_t STRIDE = (BYTES + 127) & ~(size_t)127;
};

__device__ __forceinline__ double rcp64(double y) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y));
  double e = fma(-y, r, 1.0);
  r = fma(r, e, r);
  e = fma(-y, r, 1.0);
  return fma(r, e, r);
}

// Exact u32 -> f64 on the FP64 pipe: 2^52 + x has x in its low mantissa bits.
__device__ __forceinline__ double u2d(uint32_t x) {
  return __hiloint2double(0x43300000, (int)x) - 4503599627370496.0;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}

// FMA form of the predictor, used only for the training-MAPE diagnostic.
template <int KIND>
__device__ __forceinline__ double eval_fma(const double* c, const double* inv, const double* v) {
  if constexpr (KIND == DOOLY_KIND_AFFINE) {
    return fma(c[1], v[0] * inv[0], c[0]);
  } else {
    const double f1 = v[0] * inv[0], f2 = v[1] * inv[1], f3 = v[2] * inv[2];
    double p = fma(c[1], f1, c[0]);
    p = fma(c[2], f2, p);
    p = fma(c[3], f3, p);
    p = fma(c[4], f1 * f1, p);
    p = fma(c[5], f2 * f2, p);
    p = fma(c[6], f3 * f3, p);
    p = fma(c[7], f1 * f2, p);
    p = fma(c[8], f1 * f3, p);
    return fma(c[9], f2 * f3, p);
  }
}

// Point sources -----------------------------------------------------------
template <int P>
struct GlobalPoints {
  const uint32_t* x;
  int64_t n_pts;
  const double* y;
  int64_t beg;
  __device__ __forceinline__ void load(int64_t i, uint32_t* xs, double& yv) const {
#pragma unroll
    for (int k = 0; k < P; ++k) xs[k] = __ldg(x + k * n_pts + beg + i);
    yv = __ldg(y + beg + i);
  }
};

template <int P>
struct SmemPoints {
  const uint32_t* x;  // plane 0; plane k at + k * xlen
  int xlen, xhead;
  const double* y;
  int yhead;
  __device__ __forceinline__ void load(int64_t i, uint32_t* xs, double& yv) const {
#pragma unroll
    for (int k = 0; k < P; ++k) xs[k] = x[k * xlen + xhead + (int)i];
    yv = y[yhead + (int)i];
  }
};

template <int KIND>
struct FitScratch {
  using T = FitTraits<KIND>;
  static constexpr int P = T::P, NCOL = T::NCOL, NMOM = T::NMOM;
  static constexpr int NACC = NMOM - 1 + NCOL, WARPS = T::THREADS / 32;
  double part[WARPS][NACC];
  uint32_t mn[WARPS][P], mx[WARPS][P];
  double msc[NMOM];              // scaled moments, msc[0] = n
  double b[NCOL];
  double coef[NCOL];
  double inv[P];
  uint32_t lo[P], hi[P];
  double err[WARPS];
  int8_t gidx[NCOL][NCOL];       // Gram entry -> moment index
  int8_t colmon[NCOL];           // design column -> moment index
  int8_t ex[NMOM][P];            // moment exponents
};

template <int KIND>
__device__ void write_unfitted(void* table, int64_t s, double* fit_err, uint8_t* status) {
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
}

template <int KIND>
__device__ void init_tables(FitScratch<KIND>& sh) {
  using T = FitTraits<KIND>;
  for (int t = threadIdx.x; t < T::NCOL * T::NCOL; t += blockDim.x) {
    const int i = t / T::NCOL, j = t % T::NCOL;
    if constexpr (KIND == DOOLY_KIND_AFFINE)
      sh.gidx[i][j] = (int8_t)(i + j);
    else
      sh.gidx[i][j] = kAttnGidx[i][j];
  }
  for (int t = threadIdx.x; t < T::NCOL; t += blockDim.x)
    sh.colmon[t] = KIND == DOOLY_KIND_AFFINE ? (int8_t)t : kAttnColmon[t];
  for (int t = threadIdx.x; t < T::NMOM * T::P; t += blockDim.x) {
    const int m = t / T::P, k = t % T::P;
    if constexpr (KIND == DOOLY_KIND_AFFINE)
      sh.ex[m][k] = (int8_t)m;
    else
      sh.ex[m][k] = kAttnExp[m][k];
  }
}

// Fit one signature with n >= NEED points; all threads of the CTA participate.
template <int KIND, typename Pts>
__device__ void fit_one(const Pts& pts, int64_t n, int64_t s, FitScratch<KIND>& sh, void* table,
                        double* fit_err, uint8_t* status) {
  using T = FitTraits<KIND>;
  constexpr int P = T::P, NCOL = T::NCOL, NMOM = T::NMOM, NT = T::THREADS;
  constexpr int NACC = (NMOM - 1) + NCOL, WARPS = NT / 32;
  constexpr int UNR = 4;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

  // ---------------- pass 1: raw moments + box
  constexpr int SETS = T::SETS;
  double accs[SETS][NACC];
#pragma unroll
  for (int q = 0; q < SETS; ++q)
#pragma unroll
    for (int i = 0; i < NACC; ++i) accs[q][i] = 0.0;
  uint32_t mn[P], mx[P];
#pragma unroll
  for (int k = 0; k < P; ++k) {
    mn[k] = 0xFFFFFFFFu;
    mx[k] = 0u;
  }
  for (int64_t i0 = tid; i0 < n; i0 += NT * UNR) {
    uint32_t xv[UNR][P];
    double yv[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t i = i0 + u * NT;
      if (i < n) {
        pts.load(i, xv[u], yv[u]);
      } else {
#pragma unroll
        for (int k = 0; k < P; ++k) xv[u][k] = 0u;
        yv[u] = 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (i0 + u * NT >= n) break;
      double v[P];
#pragma unroll
      for (int k = 0; k < P; ++k) {
        v[k] = u2d(xv[u][k]);
        mn[k] = min(mn[k], xv[u][k]);
        mx[k] = max(mx[k], xv[u][k]);
      }
      T::accumulate(v, yv[u], accs[u % SETS]);
    }
  }
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) {
    acc[i] = accs[0][i];
#pragma unroll
    for (int q = 1; q < SETS; ++q) acc[i] += accs[q][i];
    acc[i] = warp_sum(acc[i]);
  }
#pragma unroll
  for (int k = 0; k < P; ++k) {
    mn[k] = __reduce_min_sync(0xFFFFFFFFu, mn[k]);
    mx[k] = __reduce_max_sync(0xFFFFFFFFu, mx[k]);
  }
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) sh.part[wid][i] = acc[i];
#pragma unroll
    for (int k = 0; k < P; ++k) {
      sh.mn[wid][k] = mn[k];
      sh.mx[wid][k] = mx[k];
    }
  }
  __syncthreads();
  // ---------------- warp 0: moments -> scaled Gram -> Cholesky solve
  if (wid == 0) {
    if (lane < P) {
      uint32_t a = 0xFFFFFFFFu, b = 0u;
#pragma unroll
      for (int w = 0; w < WARPS; ++w) {
        a = min(a, sh.mn[w][lane]);
        b = max(b, sh.mx[w][lane]);
      }
      sh.lo[lane] = a;
      sh.hi[lane] = b;
      sh.inv[lane] = b > 0 ? 1.0 / (double)b : 1.0;  // IEEE division: bit-identical to the oracle
    }
    __syncwarp();
    double inv[P];
#pragma unroll
    for (int k = 0; k < P; ++k) inv[k] = sh.inv[k];
    auto scale_of = [&](int m) {
      double scl = 1.0;
#pragma unroll
      for (int k = 0; k < P; ++k)
        for (int r = 0; r < sh.ex[m][k]; ++r) scl *= inv[k];
      return scl;
    };
    for (int m = lane; m < NMOM; m += 32) {
      double raw = (double)n;
      if (m > 0) {
        raw = 0.0;
#pragma unroll
        for (int w = 0; w < WARPS; ++w) raw += sh.part[w][m - 1];
      }
      sh.msc[m] = raw * scale_of(m);
    }
    if (lane < NCOL) {
      double raw = 0.0;
#pragma unroll
      for (int w = 0; w < WARPS; ++w) raw += sh.part[w][NMOM - 1 + lane];
      sh.b[lane] = raw * scale_of(sh.colmon[lane]);
    }
    __syncwarp();
    const int r = lane < NCOL ? lane : 0;
    double g[NCOL];
#pragma unroll
    for (int k = 0; k < NCOL; ++k) g[k] = sh.msc[sh.gidx[r][k]];
    const double diag = sh.msc[sh.gidx[r][r]];
    uint32_t keep = 0;
    double rd = 0.0;  // lane j: 1 / L[j][j]
#pragma unroll
    for (int j = 0; j < NCOL; ++j) {
      const double piv = __shfl_sync(0xFFFFFFFFu, g[j], j);
      const double dj = __shfl_sync(0xFFFFFFFFu, diag, j);
      const bool kj = piv > DROP_TOL * dj;
      keep |= (uint32_t)kj << j;
      const double d = kj ? sqrt(piv) : 0.0;
      const double inv_d = kj ? rcp64(d) : 0.0;
      if (lane == j) rd = inv_d;
      double lij = lane > j ? g[j] * inv_d : 0.0;
      if (lane == j) lij = d;
      if (lane >= j) g[j] = lij;
#pragma unroll
      for (int k = j + 1; k < NCOL; ++k) {
        const double lkj = __shfl_sync(0xFFFFFFFFu, lij, k);
        g[k] = fma(-lij, lkj, g[k]);
      }
    }
    // forward: L z = b
    double t = lane < NCOL ? sh.b[lane] : 0.0, z = 0.0;
#pragma unroll
    for (int j = 0; j < NCOL; ++j) {
      const double zj = __shfl_sync(0xFFFFFFFFu, t * rd, j);  // 0 for dropped columns
      if (lane > j) t = fma(-g[j], zj, t);
      if (lane == j) z = zj;
    }
    // backward: L^T c = z
    double u = z, c = 0.0;
#pragma unroll
    for (int j = NCOL - 1; j >= 0; --j) {
      const double cj = __shfl_sync(0xFFFFFFFFu, u * rd, j);
      if (lane == j) c = cj;
#pragma unroll
      for (int m = 0; m < j; ++m) {
        const double ljm = __shfl_sync(0xFFFFFFFFu, g[m], j);  // L[j][m] from lane j
        if (lane == m) u = fma(-ljm, cj, u);
      }
    }
    (void)keep;
    if (lane < NCOL) sh.coef[lane] = c;
  }
  __syncthreads();
  // ---------------- pass 2: training MAPE with the final (clamped) predictor
  double coef[NCOL], inv[P];
#pragma unroll
  for (int i = 0; i < NCOL; ++i) coef[i] = sh.coef[i];
#pragma unroll
  for (int k = 0; k < P; ++k) inv[k] = sh.inv[k];
  double err = 0.0;
  for (int64_t i0 = tid; i0 < n; i0 += NT * UNR) {
    uint32_t xv[UNR][P];
    double yv[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t i = i0 + u * NT;
      if (i < n) {
        pts.load(i, xv[u], yv[u]);
      } else {
#pragma unroll
        for (int k = 0; k < P; ++k) xv[u][k] = 0u;
        yv[u] = 1.0;
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (i0 + u * NT >= n) break;
      double v[P];
#pragma unroll
      for (int k = 0; k < P; ++k) v[k] = u2d(xv[u][k]);
      const double p = fmax(eval_fma<KIND>(coef, inv, v), DOOLY_CLAMP_FLOOR);
      err = fma(fabs(p - yv[u]), rcp64(yv[u]), err);
    }
  }
  err = warp_sum(err);
  if (lane == 0) sh.err[wid] = err;
  __syncthreads();
  if (tid == 0) {
    double e = 0.0;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) e += sh.err[w];
    fit_err[s] = e / (double)n;
    status[s] = DOOLY_FIT_OK;
    if constexpr (KIND == DOOLY_KIND_AFFINE) {
      dooly_affine_row* row = static_cast<dooly_affine_row*>(table) + s;
      row->c0 = coef[0];
      row->c1 = coef[1];
      row->inv_scale = inv[0];
      row->lo = sh.lo[0];
      row->hi = sh.hi[0];
    } else {
      dooly_attn_row* row = static_cast<dooly_attn_row*>(table) + s;
      for (int i = 0; i < 10; ++i) row->c[i] = coef[i];
      for (int k = 0; k < 3; ++k) {
        row->inv_scale[k] = inv[k];
        row->lo[k] = sh.lo[k];
        row->hi[k] = sh.hi[k];
      }
    }
  }
  // the caller's next __syncthreads (or the next signature's first one)
  // orders these smem reads before any rewrite of sh
}

// --------------------------------------------------------------- bulk copies
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct Window {  // aligned bulk window of elements [beg, end) of an array
  int64_t abeg;  // aligned-down first element copied
  int64_t aend;  // end of the bulk-copied range (aligned)
  int head;      // beg - abeg
};

__device__ __forceinline__ Window make_window(int64_t beg, int64_t end, int64_t n_total,
                                              int per16) {
  Window w;
  w.abeg = beg / per16 * per16;
  int64_t e = (end + per16 - 1) / per16 * per16;
  const int64_t cap = n_total / per16 * per16;  // never read past the array
  w.aend = e < cap ? e : cap;
  if (w.aend < w.abeg) w.aend = w.abeg;
  w.head = (int)(beg - w.abeg);
  return w;
}

// Issue the bulk copies of one signature into a stage; the (<4) tail elements
// past the last aligned chunk of the arrays are loaded by the consumers.
template <int KIND>
__device__ void issue_stage(unsigned char* stage, uint64_t* bar, const uint32_t* x, int64_t n_pts,
                            const double* y, int64_t beg, int64_t end) {
  using S = Stage<KIND>;
  const Window wy = make_window(beg, end, n_pts, 2);
  const Window wx = make_window(beg, end, n_pts, 4);
  const uint32_t by = (uint32_t)((wy.aend - wy.abeg) * 8);
  const uint32_t bx = (uint32_t)((wx.aend - wx.abeg) * 4);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  mbar_expect_tx(bar, by + S::P * bx);
  double* sy = reinterpret_cast<double*>(stage);
  uint32_t* sx = reinterpret_cast<uint32_t*>(stage + (size_t)S::Y_LEN * 8);
  if (by) bulk_g2s(sy, y + wy.abeg, by, bar);
  if (bx)
    for (int k = 0; k < S::P; ++k) bulk_g2s(sx + k * S::X_LEN, x + k * n_pts + wx.abeg, bx, bar);
}

template <int KIND>
__global__ void __launch_bounds__(FitTraits<KIND>::THREADS, FIT_CTAS_PER_SM) fit_bulk_kernel(
    const uint32_t* __restrict__ x, int64_t n_pts, const double* __restrict__ y,
    const int64_t* __restrict__ off, int64_t n_sig, void* __restrict__ table,
    double* __restrict__ fit_err, uint8_t* __restrict__ status, bool bulk_ok, int nst) {
  using T = FitTraits<KIND>;
  using S = Stage<KIND>;
  const int NST = nst;  // 1..4 stages (runtime: tuned per kind at launch)
  extern __shared__ __align__(128) unsigned char dyn[];
  __shared__ __align__(8) uint64_t bars[4];
  __shared__ FitScratch<KIND> sh;
  const int tid = threadIdx.x;

  // signatures of this CTA: s_k = blockIdx.x + k * gridDim.x
  auto sig_of = [&](int64_t k) { return (int64_t)blockIdx.x + k * (int64_t)gridDim.x; };
  auto stageable = [&](int64_t s) {
    const int64_t n = off[s + 1] - off[s];
    return bulk_ok && n >= T::NEED && n <= FIT_CAP;
  };
  init_tables<KIND>(sh);
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int k = 0; k < NST - 1; ++k) {
      const int64_t s = sig_of(k);
      if (s < n_sig && stageable(s))
        issue_stage<KIND>(dyn + (size_t)k * S::STRIDE, &bars[k], x, n_pts, y, off[s], off[s + 1]);
    }
  }
  // CSR offsets are software-pipelined two signatures ahead so their global
  // load latency never sits on the critical path (ncu: the refill's dependent
  // off[] loads were stalling the whole CTA at the next barrier).
  auto load_off = [&](int64_t kk, int64_t& b, int64_t& e) {
    const int64_t ss = sig_of(kk);
    b = ss < n_sig ? __ldg(off + ss) : 0;
    e = ss < n_sig ? __ldg(off + ss + 1) : 0;
  };
  int64_t ob[4], oe[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) load_off(i, ob[i], oe[i]);
  auto stageable_be = [&](int64_t b, int64_t e) {
    return bulk_ok && e - b >= T::NEED && e - b <= FIT_CAP;
  };
  uint32_t phase_bits = 0;  // per-stage parity
  for (int64_t k = 0;; ++k) {
    const int64_t s = sig_of(k);
    if (s >= n_sig) break;
    const int64_t beg = ob[0], end = oe[0], n = end - beg;
    // keep STAGES-1 signatures ahead: refill the stage freed by signature k-1
    if (tid == 0) {
      const int64_t kn = k + NST - 1;
      const int64_t sn = sig_of(kn);
      const int64_t nb = NST == 1 ? ob[0] : NST == 2 ? ob[1] : NST == 3 ? ob[2] : ob[3];
      const int64_t ne = NST == 1 ? oe[0] : NST == 2 ? oe[1] : NST == 3 ? oe[2] : oe[3];
      if (sn < n_sig && stageable_be(nb, ne)) {
        const int st = (int)(kn % NST);
        issue_stage<KIND>(dyn + (size_t)st * S::STRIDE, &bars[st], x, n_pts, y, nb, ne);
      }
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      ob[i] = ob[i + 1];
      oe[i] = oe[i + 1];
    }
    load_off(k + 4, ob[3], oe[3]);
    if (n < T::NEED) {
      if (tid == 0) write_unfitted<KIND>(table, s, fit_err, status);
      continue;  // no stage was used (stageable() is false)
    }
    if (!stageable_be(beg, end)) {  // oversized / unaligned inputs: stream from global memory
      GlobalPoints<T::P> gp{x, n_pts, y, beg};
      fit_one<KIND>(gp, n, s, sh, table, fit_err, status);
      __syncthreads();
      continue;
    }
    const int st = (int)(k % NST);
    unsigned char* stage = dyn + (size_t)st * S::STRIDE;
    mbar_wait(&bars[st], (phase_bits >> st) & 1u);
    phase_bits ^= 1u << st;
    const Window wy = make_window(beg, end, n_pts, 2);
    const Window wx = make_window(beg, end, n_pts, 4);
    double* sy = reinterpret_cast<double*>(stage);
    uint32_t* sx = reinterpret_cast<uint32_t*>(stage + (size_t)S::Y_LEN * 8);
    // tail elements past the last aligned chunk of the arrays (end of the data only)
    if (tid < 4) {
      const int64_t j = wx.aend + tid;
      if (j < end)
        for (int kk = 0; kk < T::P; ++kk) sx[kk * S::X_LEN + (j - wx.abeg)] = x[kk * n_pts + j];
      const int64_t jy = wy.aend + tid;
      if (jy < end) sy[jy - wy.abeg] = y[jy];
    }
    __syncthreads();
    SmemPoints<T::P> sp{sx, S::X_LEN, wx.head, sy, wy.head};
    fit_one<KIND>(sp, n, s, sh, table, fit_err, status);
    __syncthreads();  // stage and scratch free for reuse
  }
}

template <int KIND>
static cudaError_t launch_kind(const uint32_t* x, int64_t n_pts, const double* y,
                               const int64_t* off, int64_t n_sig, void* table, double* fit_err,
                               uint8_t* status, cudaStream_t stream, int n_sm) {
  int nst = FitTraits<KIND>::STAGES;
  if (const char* env = getenv(KIND == DOOLY_KIND_AFFINE ? "DOOLY_FIT_STAGES_AFFINE"
                                                         : "DOOLY_FIT_STAGES_ATTN")) {
    const int v = atoi(env);  // tuning knob (profiles/); 1..4
    if (v >= 1 && v <= 4) nst = v;
  }
  const size_t smem = (size_t)nst * Stage<KIND>::STRIDE;
  cudaError_t e = cudaFuncSetAttribute(fit_bulk_kernel<KIND>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // 1-D TMA needs 16-B aligned sources: plane bases and the y array
  const bool bulk_ok = ((uintptr_t)x % 16 == 0) && ((uintptr_t)y % 16 == 0) &&
                       (FitTraits<KIND>::P == 1 || n_pts % 4 == 0);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fit_bulk_kernel<KIND>,
                                                FitTraits<KIND>::THREADS, smem);
  int64_t blocks = (int64_t)n_sm * (per_sm > 0 ? per_sm : 1);
  if (blocks > n_sig) blocks = n_sig;
  fit_bulk_kernel<KIND><<<(unsigned)blocks, FitTraits<KIND>::THREADS, smem, stream>>>(
      x, n_pts, y, off, n_sig, table, fit_err, status, bulk_ok, nst);
  return cudaGetLastError();
}

cudaError_t launch_fit(int kind, const uint32_t* x, int64_t n_pts, const double* y,
                       const int64_t* off, int64_t n_sig, void* table, double* fit_err,
                       uint8_t* status, cudaStream_t stream, int n_sm) {
  if (n_sig == 0) return cudaSuccess;
  if (kind == DOOLY_KIND_AFFINE)
    return launch_kind<DOOLY_KIND_AFFINE>(x, n_pts, y, off, n_sig, table, fit_err, status,
                                          stream, n_sm);
  return launch_kind<DOOLY_KIND_ATTN>(x, n_pts, y, off, n_sig, table, fit_err, status, stream,
                                      n_sm);
}

}  // namespace dooly
