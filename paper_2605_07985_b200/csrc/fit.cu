// K2 — batched per-signature least-squares fit (replaces fit).
//
// Data path (B200): a persistent kernel, several 128-thread CTAs per SM (4 for
// affine, 2 for attention: the shared-memory stage is the limiter).  Each CTA
// owns one stage that holds a whole signature (<= 4096 points) as two halves
// of <= 2048 points, each filled by the bulk-copy (1-D TMA) engine
// (`cp.async.bulk` + mbarrier complete_tx).  Both passes over a signature read
// shared memory, so every point crosses HBM exactly once.  The halves are
// refilled as soon as pass 2 has finished with them: the first half of the
// next signature streams in underneath the second half of pass 2, the second
// half underneath the write-out and the next signature's first-half pass 1.
// (A finer chunk ring with a thread-0 producer was measured and was slower:
// the per-chunk bookkeeping and producer imbalance cost more than the extra
// overlap bought — profiles/r1_ncu_summary.md.)  Signatures larger than a
// stage, or unaligned inputs, use a direct global-memory path with the same
// arithmetic.
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
#include "attn_moments.cuh"
#include <stdlib.h>
#include <string.h>

#include "common.cuh"

namespace dooly {

constexpr double DROP_TOL = 1e-9;
constexpr int FIT_THREADS = 128;
constexpr int FIT_WARPS = FIT_THREADS / 32;
constexpr int FIT_UNR = 4;
constexpr int FIT_HALF = 2048;  // points per half stage; a stage holds 2 * FIT_HALF

template <int KIND>
struct FitTraits;

template <>
struct FitTraits<DOOLY_KIND_AFFINE> {
  static constexpr int P = 1;      // features
  static constexpr int NCOL = 2;   // design columns [1, f]
  static constexpr int NMOM = 3;   // 1, x, x^2
  static constexpr int NEED = 4;   // max(4, NCOL + 1)   (App. A.8)
  static constexpr int SETS = 2;   // independent accumulator sets (breaks DADD chains)
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
  static constexpr int SETS = 1;   // 44 independent accumulators already give the ILP
  __device__ static __forceinline__ void accumulate(const double* v, double y, double* acc) {
    attn_accumulate(v[0], v[1], v[2], y, acc);
  }
};

// Half-stage layout: y[FIT_HALF + 2] f64, then P planes of x[FIT_HALF + 4] u32
// (the +2/+4 hold the head misalignment of the aligned bulk window).
template <int KIND>
struct Half {
  static constexpr int P = FitTraits<KIND>::P;
  static constexpr int Y_LEN = FIT_HALF + 2;
  static constexpr int X_LEN = FIT_HALF + 4;
  static constexpr size_t BYTES = (size_t)Y_LEN * 8 + (size_t)P * X_LEN * 4;
  static constexpr size_t STRIDE = (BYTES + 127) & ~(size_t)127;
  static constexpr size_t STAGE_BYTES = 2 * STRIDE;
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

// Point sources ----------------------------------------------------------
template <int P>
struct GlobalPoints {  // points beg + i of the CSR arrays
  const uint32_t* x;
  int64_t n_pts;
  const double* y;
  int64_t beg;
  __device__ __forceinline__ void load(int i, uint32_t* xs, double& yv) const {
#pragma unroll
    for (int k = 0; k < P; ++k) xs[k] = __ldg(x + k * n_pts + beg + i);
    yv = __ldg(y + beg + i);
  }
};

template <int P>
struct HalfPoints {  // one half stage; points past the bulk window come from global
  const uint32_t* sx;
  int xlen, xhead, xbulk;  // xbulk: points served from smem
  const double* sy;
  int yhead, ybulk;
  GlobalPoints<P> g;       // global fallback for the (<4) array-end tail points
  __device__ __forceinline__ void load(int i, uint32_t* xs, double& yv) const {
    if (i < xbulk) {
#pragma unroll
      for (int k = 0; k < P; ++k) xs[k] = sx[k * xlen + xhead + i];
    } else {
#pragma unroll
      for (int k = 0; k < P; ++k) xs[k] = __ldg(g.x + k * g.n_pts + g.beg + i);
    }
    yv = i < ybulk ? sy[yhead + i] : __ldg(g.y + g.beg + i);
  }
  // Whole half in shared memory with 16-B aligned windows: 4-point vector loads.
  __device__ __forceinline__ bool dense(int cnt) const {
    return xhead == 0 && yhead == 0 && xbulk >= cnt && ybulk >= cnt;
  }
  __device__ __forceinline__ void load4(int i4, uint32_t (*xs)[P], double* yv) const {
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const uint4 v = *reinterpret_cast<const uint4*>(sx + k * xlen + i4);
      xs[0][k] = v.x;
      xs[1][k] = v.y;
      xs[2][k] = v.z;
      xs[3][k] = v.w;
    }
    const double2 a = *reinterpret_cast<const double2*>(sy + i4);
    const double2 b = *reinterpret_cast<const double2*>(sy + i4 + 2);
    yv[0] = a.x;
    yv[1] = a.y;
    yv[2] = b.x;
    yv[3] = b.y;
  }
};

template <int KIND>
struct FitScratch {
  using T = FitTraits<KIND>;
  static constexpr int P = T::P, NCOL = T::NCOL, NMOM = T::NMOM;
  static constexpr int NACC = NMOM - 1 + NCOL;
  double part[FIT_WARPS][NACC];
  uint32_t mn[FIT_WARPS][P], mx[FIT_WARPS][P];
  double msc[NMOM];              // scaled moments, msc[0] = n
  double b[NCOL];
  double coef[NCOL];
  double inv[P];
  uint32_t lo[P], hi[P];
  double err[FIT_WARPS];
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

// --------------------------------------------------------------- fit phases
template <int KIND>
struct Pass1State {
  static constexpr int NACC = FitTraits<KIND>::NMOM - 1 + FitTraits<KIND>::NCOL;
  double accs[FitTraits<KIND>::SETS][NACC];
  uint32_t mn[FitTraits<KIND>::P], mx[FitTraits<KIND>::P];
  __device__ __forceinline__ void reset() {
#pragma unroll
    for (int q = 0; q < FitTraits<KIND>::SETS; ++q)
#pragma unroll
      for (int i = 0; i < NACC; ++i) accs[q][i] = 0.0;
#pragma unroll
    for (int k = 0; k < FitTraits<KIND>::P; ++k) {
      mn[k] = 0xFFFFFFFFu;
      mx[k] = 0u;
    }
  }
};

// Accumulate points [0, cnt) of a source (threads stride over them).
template <int KIND, typename Pts>
__device__ __forceinline__ void pass1(const Pts& pts, int cnt, Pass1State<KIND>& st) {
  using T = FitTraits<KIND>;
  constexpr int P = T::P;
  for (int i0 = threadIdx.x; i0 < cnt; i0 += FIT_THREADS * FIT_UNR) {
    uint32_t xv[FIT_UNR][P];
    double yv[FIT_UNR];
#pragma unroll
    for (int u = 0; u < FIT_UNR; ++u) {
      const int i = i0 + u * FIT_THREADS;
      if (i < cnt) {
        pts.load(i, xv[u], yv[u]);
      } else {
#pragma unroll
        for (int k = 0; k < P; ++k) xv[u][k] = 0u;
        yv[u] = 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < FIT_UNR; ++u) {
      if (i0 + u * FIT_THREADS >= cnt) break;
      double v[P];
#pragma unroll
      for (int k = 0; k < P; ++k) {
        v[k] = u2d(xv[u][k]);
        st.mn[k] = min(st.mn[k], xv[u][k]);
        st.mx[k] = max(st.mx[k], xv[u][k]);
      }
      T::accumulate(v, yv[u], st.accs[u % T::SETS]);
    }
  }
}

template <int KIND>
__device__ __forceinline__ void pass1_point(const uint32_t* xv, double yv, Pass1State<KIND>& st,
                                            int set) {
  constexpr int P = FitTraits<KIND>::P;
  double v[P];
#pragma unroll
  for (int k = 0; k < P; ++k) {
    v[k] = u2d(xv[k]);
    st.mn[k] = min(st.mn[k], xv[k]);
    st.mx[k] = max(st.mx[k], xv[k]);
  }
  FitTraits<KIND>::accumulate(v, yv, st.accs[set]);
}

// Half-stage pass 1: each thread takes 4 consecutive points with 16-B smem
// loads when the half is dense and aligned, else the generic strided loop.
template <int KIND>
__device__ __forceinline__ void pass1_half(const HalfPoints<FitTraits<KIND>::P>& hp, int cnt,
                                           Pass1State<KIND>& st) {
  constexpr int P = FitTraits<KIND>::P, SETS = FitTraits<KIND>::SETS;
  if (!hp.dense(cnt)) {
    pass1<KIND>(hp, cnt, st);
    return;
  }
  for (int i4 = 4 * threadIdx.x; i4 < cnt; i4 += 4 * FIT_THREADS) {
    if (i4 + 4 <= cnt) {
      uint32_t xv[4][P];
      double yv[4];
      hp.load4(i4, xv, yv);
#pragma unroll
      for (int u = 0; u < 4; ++u) pass1_point<KIND>(xv[u], yv[u], st, u % SETS);
    } else {
      for (int i = i4; i < cnt; ++i) {
        uint32_t xv[P];
        double yv;
        hp.load(i, xv, yv);
        pass1_point<KIND>(xv, yv, st, 0);
      }
    }
  }
}

// Reduce pass-1 state, solve (warp 0); on return sh.coef/inv/lo/hi are valid
// for every thread (ends with __syncthreads).
template <int KIND>
__device__ void reduce_and_solve(Pass1State<KIND>& st, int64_t n, FitScratch<KIND>& sh) {
  using T = FitTraits<KIND>;
  constexpr int P = T::P, NCOL = T::NCOL, NMOM = T::NMOM;
  constexpr int NACC = (NMOM - 1) + NCOL;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
#pragma unroll
  for (int i = 0; i < NACC; ++i) {
    double a = st.accs[0][i];
#pragma unroll
    for (int q = 1; q < T::SETS; ++q) a += st.accs[q][i];
    a = warp_sum(a);
    if (lane == 0) sh.part[wid][i] = a;
  }
#pragma unroll
  for (int k = 0; k < P; ++k) {
    const uint32_t a = __reduce_min_sync(0xFFFFFFFFu, st.mn[k]);
    const uint32_t b = __reduce_max_sync(0xFFFFFFFFu, st.mx[k]);
    if (lane == 0) {
      sh.mn[wid][k] = a;
      sh.mx[wid][k] = b;
    }
  }
  __syncthreads();
  if (wid == 0) {
    if (lane < P) {
      uint32_t a = 0xFFFFFFFFu, b = 0u;
#pragma unroll
      for (int w = 0; w < FIT_WARPS; ++w) {
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
        for (int w = 0; w < FIT_WARPS; ++w) raw += sh.part[w][m - 1];
      }
      sh.msc[m] = raw * scale_of(m);
    }
    if (lane < NCOL) {
      double raw = 0.0;
#pragma unroll
      for (int w = 0; w < FIT_WARPS; ++w) raw += sh.part[w][NMOM - 1 + lane];
      sh.b[lane] = raw * scale_of(sh.colmon[lane]);
    }
    __syncwarp();
    const int r = lane < NCOL ? lane : 0;
    double g[NCOL];
#pragma unroll
    for (int k = 0; k < NCOL; ++k) g[k] = sh.msc[sh.gidx[r][k]];
    const double diag = sh.msc[sh.gidx[r][r]];
    double rd = 0.0;  // lane j: 1 / L[j][j] (0 for a dropped column)
#pragma unroll
    for (int j = 0; j < NCOL; ++j) {
      const double piv = __shfl_sync(0xFFFFFFFFu, g[j], j);
      const double dj = __shfl_sync(0xFFFFFFFFu, diag, j);
      const bool kj = piv > DROP_TOL * dj;
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
      const double zj = __shfl_sync(0xFFFFFFFFu, t * rd, j);
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
    if (lane < NCOL) sh.coef[lane] = c;
  }
  __syncthreads();
}

template <int KIND, typename Pts>
__device__ __forceinline__ void pass2(const Pts& pts, int cnt, const double* coef,
                                      const double* inv, double& err) {
  constexpr int P = FitTraits<KIND>::P;
  for (int i0 = threadIdx.x; i0 < cnt; i0 += FIT_THREADS * FIT_UNR) {
    uint32_t xv[FIT_UNR][P];
    double yv[FIT_UNR];
#pragma unroll
    for (int u = 0; u < FIT_UNR; ++u) {
      const int i = i0 + u * FIT_THREADS;
      if (i < cnt) {
        pts.load(i, xv[u], yv[u]);
      } else {
#pragma unroll
        for (int k = 0; k < P; ++k) xv[u][k] = 0u;
        yv[u] = 1.0;
      }
    }
#pragma unroll
    for (int u = 0; u < FIT_UNR; ++u) {
      if (i0 + u * FIT_THREADS >= cnt) break;
      double v[P];
#pragma unroll
      for (int k = 0; k < P; ++k) v[k] = u2d(xv[u][k]);
      const double p = fmax(eval_fma<KIND>(coef, inv, v), DOOLY_CLAMP_FLOOR);
      err = fma(fabs(p - yv[u]), rcp64(yv[u]), err);
    }
  }
}

template <int KIND>
__device__ __forceinline__ double mape_term(const uint32_t* xv, double yv, const double* coef,
                                            const double* inv) {
  constexpr int P = FitTraits<KIND>::P;
  double v[P];
#pragma unroll
  for (int k = 0; k < P; ++k) v[k] = u2d(xv[k]);
  const double p = fmax(eval_fma<KIND>(coef, inv, v), DOOLY_CLAMP_FLOOR);
  return fabs(p - yv) * rcp64(yv);
}

template <int KIND>
__device__ __forceinline__ void pass2_half(const HalfPoints<FitTraits<KIND>::P>& hp, int cnt,
                                           const double* coef, const double* inv, double& err) {
  constexpr int P = FitTraits<KIND>::P;
  if (!hp.dense(cnt)) {
    pass2<KIND>(hp, cnt, coef, inv, err);
    return;
  }
  double e2 = 0.0;
  for (int i4 = 4 * threadIdx.x; i4 < cnt; i4 += 4 * FIT_THREADS) {
    if (i4 + 4 <= cnt) {
      uint32_t xv[4][P];
      double yv[4];
      hp.load4(i4, xv, yv);
      err += mape_term<KIND>(xv[0], yv[0], coef, inv);
      e2 += mape_term<KIND>(xv[1], yv[1], coef, inv);
      err += mape_term<KIND>(xv[2], yv[2], coef, inv);
      e2 += mape_term<KIND>(xv[3], yv[3], coef, inv);
    } else {
      for (int i = i4; i < cnt; ++i) {
        uint32_t xv[P];
        double yv;
        hp.load(i, xv, yv);
        err += mape_term<KIND>(xv, yv, coef, inv);
      }
    }
  }
  err += e2;
}

// Reduce the MAPE and write the row (ends with __syncthreads).
template <int KIND>
__device__ void finish(double err, int64_t n, int64_t s, FitScratch<KIND>& sh, void* table,
                       double* fit_err, uint8_t* status) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  err = warp_sum(err);
  if (lane == 0) sh.err[wid] = err;
  __syncthreads();
  if (tid == 0) {
    double e = 0.0;
#pragma unroll
    for (int w = 0; w < FIT_WARPS; ++w) e += sh.err[w];
    fit_err[s] = e / (double)n;
    status[s] = DOOLY_FIT_OK;
    if constexpr (KIND == DOOLY_KIND_AFFINE) {
      dooly_affine_row* row = static_cast<dooly_affine_row*>(table) + s;
      row->c0 = sh.coef[0];
      row->c1 = sh.coef[1];
      row->inv_scale = sh.inv[0];
      row->lo = sh.lo[0];
      row->hi = sh.hi[0];
    } else {
      dooly_attn_row* row = static_cast<dooly_attn_row*>(table) + s;
      for (int i = 0; i < 10; ++i) row->c[i] = sh.coef[i];
      for (int k = 0; k < 3; ++k) {
        row->inv_scale[k] = sh.inv[k];
        row->lo[k] = sh.lo[k];
        row->hi[k] = sh.hi[k];
      }
    }
  }
  __syncthreads();
}

// --------------------------------------------------------------- mbarriers
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
  int64_t aend;  // end of the bulk-copied range (aligned, never past the array)
  int head;      // beg - abeg
};

__device__ __forceinline__ Window make_window(int64_t beg, int64_t end, int64_t n_total,
                                              int per16) {
  Window w;
  w.abeg = beg / per16 * per16;
  const int64_t e = (end + per16 - 1) / per16 * per16;
  const int64_t cap = n_total / per16 * per16;
  w.aend = e < cap ? e : cap;
  if (w.aend < w.abeg) w.aend = w.abeg;
  w.head = (int)(beg - w.abeg);
  return w;
}

// Issue points [c0, c1) into one half stage (thread 0).
template <int KIND>
__device__ void issue_half(unsigned char* half, uint64_t* bar, const uint32_t* x, int64_t n_pts,
                           const double* y, int64_t c0, int64_t c1) {
  using H = Half<KIND>;
  const Window wy = make_window(c0, c1, n_pts, 2);
  const Window wx = make_window(c0, c1, n_pts, 4);
  const uint32_t by = (uint32_t)((wy.aend - wy.abeg) * 8);
  const uint32_t bx = (uint32_t)((wx.aend - wx.abeg) * 4);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  mbar_expect_tx(bar, by + H::P * bx);
  if (by) bulk_g2s(half, y + wy.abeg, by, bar);
  if (bx) {
    uint32_t* sx = reinterpret_cast<uint32_t*>(half + (size_t)H::Y_LEN * 8);
    for (int k = 0; k < H::P; ++k) bulk_g2s(sx + k * H::X_LEN, x + k * n_pts + wx.abeg, bx, bar);
  }
}

template <int KIND>
__device__ __forceinline__ HalfPoints<FitTraits<KIND>::P> half_points(
    unsigned char* half, const uint32_t* x, int64_t n_pts, const double* y, int64_t c0,
    int64_t c1) {
  using H = Half<KIND>;
  const Window wy = make_window(c0, c1, n_pts, 2);
  const Window wx = make_window(c0, c1, n_pts, 4);
  return HalfPoints<FitTraits<KIND>::P>{
      reinterpret_cast<const uint32_t*>(half + (size_t)H::Y_LEN * 8), H::X_LEN, wx.head,
      (int)(wx.aend - c0), reinterpret_cast<const double*>(half), wy.head, (int)(wy.aend - c0),
      GlobalPoints<FitTraits<KIND>::P>{x, n_pts, y, c0}};
}

template <int KIND>
__global__ void __launch_bounds__(FIT_THREADS) fit_stage_kernel(
    const uint32_t* __restrict__ x, int64_t n_pts, const double* __restrict__ y,
    const int64_t* __restrict__ off, int64_t n_sig, void* __restrict__ table,
    double* __restrict__ fit_err, uint8_t* __restrict__ status, bool bulk_ok) {
  using T = FitTraits<KIND>;
  using H = Half<KIND>;
  extern __shared__ __align__(128) unsigned char dyn[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ FitScratch<KIND> sh;
  const int tid = threadIdx.x;
  unsigned char* const half0 = dyn;
  unsigned char* const half1 = dyn + H::STRIDE;

  auto sig_of = [&](int64_t k) { return (int64_t)blockIdx.x + k * (int64_t)gridDim.x; };
  auto staged = [&](int64_t b, int64_t e) {
    return bulk_ok && e - b >= T::NEED && e - b <= 2 * FIT_HALF;
  };
  auto split = [](int64_t b, int64_t e) { return e - b < FIT_HALF ? e - b : (int64_t)FIT_HALF; };

  init_tables<KIND>(sh);
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // CSR offsets software-pipelined two signatures ahead (all threads)
  auto load_off = [&](int64_t kk, int64_t& b, int64_t& e) {
    const int64_t ss = sig_of(kk);
    b = ss < n_sig ? __ldg(off + ss) : 0;
    e = ss < n_sig ? __ldg(off + ss + 1) : 0;
  };
  int64_t cb, ce, nb, ne, nnb, nne;
  load_off(0, cb, ce);
  load_off(1, nb, ne);
  load_off(2, nnb, nne);
  // producer (thread 0): the first signature's halves
  if (tid == 0 && sig_of(0) < n_sig && staged(cb, ce)) {
    const int64_t pa = split(cb, ce);
    issue_half<KIND>(half0, &bar[0], x, n_pts, y, cb, cb + pa);
    if (ce - cb > pa) issue_half<KIND>(half1, &bar[1], x, n_pts, y, cb + pa, ce);
  }
  uint32_t par0 = 0u, par1 = 0u;
  Pass1State<KIND> st;
  for (int64_t k = 0;; ++k) {
    const int64_t s = sig_of(k);
    if (s >= n_sig) break;
    const int64_t beg = cb, end = ce, n = end - beg;
    const int64_t nbeg = nb, nend = ne;
    const bool next_staged = sig_of(k + 1) < n_sig && staged(nbeg, nend);
    const int64_t npa = next_staged ? split(nbeg, nend) : 0;
    cb = nb;
    ce = ne;
    nb = nnb;
    ne = nne;
    load_off(k + 3, nnb, nne);

    if (!staged(beg, end)) {
      // halves unused by this signature: start the next one's loads right away
      if (tid == 0 && next_staged) {
        issue_half<KIND>(half0, &bar[0], x, n_pts, y, nbeg, nbeg + npa);
        if (nend - nbeg > npa) issue_half<KIND>(half1, &bar[1], x, n_pts, y, nbeg + npa, nend);
      }
      if (n < T::NEED) {
        if (tid == 0) write_unfitted<KIND>(table, s, fit_err, status);
        continue;
      }
      st.reset();  // oversized / unaligned: direct global path
      const GlobalPoints<T::P> gp{x, n_pts, y, beg};
      pass1<KIND>(gp, (int)n, st);
      reduce_and_solve<KIND>(st, n, sh);
      double err = 0.0;
      pass2<KIND>(gp, (int)n, sh.coef, sh.inv, err);
      finish<KIND>(err, n, s, sh, table, fit_err, status);
      continue;
    }
    const int64_t pa = split(beg, end);
    const bool has_b = n > pa;
    const auto ha = half_points<KIND>(half0, x, n_pts, y, beg, beg + pa);
    const auto hb = half_points<KIND>(half1, x, n_pts, y, beg + pa, end);
    // ---- pass 1, half by half as they land
    st.reset();
    mbar_wait(&bar[0], par0);
    par0 ^= 1u;
    pass1_half<KIND>(ha, (int)pa, st);
    if (has_b) {
      mbar_wait(&bar[1], par1);
      par1 ^= 1u;
      pass1_half<KIND>(hb, (int)(n - pa), st);
    }
    reduce_and_solve<KIND>(st, n, sh);
    double coef[T::NCOL], inv[T::P];
#pragma unroll
    for (int i = 0; i < T::NCOL; ++i) coef[i] = sh.coef[i];
#pragma unroll
    for (int kk = 0; kk < T::P; ++kk) inv[kk] = sh.inv[kk];
    // ---- pass 2; each half is refilled with the next signature once released
    double err = 0.0;
    pass2_half<KIND>(ha, (int)pa, coef, inv, err);
    __syncthreads();  // half 0 free
    if (tid == 0 && next_staged) issue_half<KIND>(half0, &bar[0], x, n_pts, y, nbeg, nbeg + npa);
    if (has_b) pass2_half<KIND>(hb, (int)(n - pa), coef, inv, err);
    finish<KIND>(err, n, s, sh, table, fit_err, status);  // ends with __syncthreads: half 1 free
    if (tid == 0 && next_staged && nend - nbeg > npa)
      issue_half<KIND>(half1, &bar[1], x, n_pts, y, nbeg + npa, nend);
  }
}

template <int KIND>
static cudaError_t launch_kind(const uint32_t* x, int64_t n_pts, const double* y,
                               const int64_t* off, int64_t n_sig, void* table, double* fit_err,
                               uint8_t* status, cudaStream_t stream, int n_sm) {
  const size_t smem = Half<KIND>::STAGE_BYTES;
  cudaError_t e = cudaFuncSetAttribute(fit_stage_kernel<KIND>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // 1-D TMA needs 16-B aligned sources: plane bases and the y array
  const bool bulk_ok = ((uintptr_t)x % 16 == 0) && ((uintptr_t)y % 16 == 0) &&
                       (FitTraits<KIND>::P == 1 || n_pts % 4 == 0);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fit_stage_kernel<KIND>, FIT_THREADS,
                                                smem);
  int64_t blocks = (int64_t)n_sm * (per_sm > 0 ? per_sm : 1);
  if (blocks > n_sig) blocks = n_sig;
  fit_stage_kernel<KIND><<<(unsigned)blocks, FIT_THREADS, smem, stream>>>(
      x, n_pts, y, off, n_sig, table, fit_err, status, bulk_ok);
  return cudaGetLastError();
}

// ====================================================================
// Affine CSR path, one WARP per signature (the default for affine).  Pass 1
// streams the signature's x (u32) and y (f64) from HBM, 4 consecutive points
// per lane per step with 16-B / 32-B vector loads (4 steps in flight),
// tagged L2::evict_last; the raw sums (x, x^2, y, xy; two accumulator sets)
// and the box reduce with shuffles; every lane solves the 2x2 scaled normal
// equations with the same Cholesky-with-drop arithmetic as reduce_and_solve;
// pass 2 re-streams the points — normally L2 hits — for the training MAPE.
// No shared memory and no CTA barrier: every warp streams independently,
// where the staged CTA kernel stops a whole CTA at each signature's solve.
// x planes (16 B per lane step): L2 eviction hints need 256-bit accesses, so
// x goes through the default policy (16 KB per 4096-point signature).
__device__ __forceinline__ uint4 ld_keep_u4(const void* p, bool) { return ld_stream_u4(p); }
__device__ __forceinline__ double4 ld_keep_d4(const double* p, bool keep) {
  double4 v;
  if (keep)
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_last.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  else
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}

// Visit points [beg, beg + n) of a signature once: the misaligned head and the
// tail point by point, the aligned body 4 points per lane with FA_YS steps of
// loads issued ahead of their use.
constexpr int FA_YS = 4;
template <typename F4, typename F1>
__device__ __forceinline__ void warp_stream_affine(const uint32_t* x, const double* y, int64_t beg,
                                                   int64_t n, bool vec, bool keep, F4&& f4,
                                                   F1&& f1) {
  const int lane = threadIdx.x & 31;
  int64_t h = vec ? (4 - (beg & 3)) & 3 : 0;  // head points before the 32-B aligned body
  if (h > n) h = n;
  if (lane < h) f1(__ldg(x + beg + lane), __ldg(y + beg + lane));
  int64_t i = h;
  if (vec) {
    const int64_t body = h + (n - h) / 128 * 128;
    for (; i + 128 * FA_YS <= body; i += 128 * FA_YS) {
      uint4 xv[FA_YS];
      double4 yv[FA_YS];
#pragma unroll
      for (int t = 0; t < FA_YS; ++t) {
        const int64_t q = beg + i + 128 * t + 4 * lane;
        xv[t] = ld_keep_u4(x + q, keep);
        yv[t] = ld_keep_d4(y + q, keep);
      }
#pragma unroll
      for (int t = 0; t < FA_YS; ++t) f4(xv[t], yv[t]);
    }
    for (; i < body; i += 128) {
      const int64_t q = beg + i + 4 * lane;
      f4(ld_keep_u4(x + q, keep), ld_keep_d4(y + q, keep));
    }
  }
  for (int64_t k = i + lane; k < n; k += 32) f1(__ldg(x + beg + k), __ldg(y + beg + k));
}

__global__ void __launch_bounds__(256, 2) fit_affine_warp_kernel(
    const uint32_t* __restrict__ x, const double* __restrict__ y, const int64_t* __restrict__ off,
    int64_t n_sig, dooly_affine_row* __restrict__ table, double* __restrict__ fit_err,
    uint8_t* __restrict__ status, bool vec_ok) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = warp; s < n_sig; s += n_warps) {
    const int64_t beg = __ldg(off + s), n = __ldg(off + s + 1) - beg;
    if (n < FitTraits<DOOLY_KIND_AFFINE>::NEED) {
      if (lane == 0) write_unfitted<DOOLY_KIND_AFFINE>(table, s, fit_err, status);
      continue;
    }
    // ---- pass 1: raw sums (x, x^2, y, xy) in two sets, and the box
    double a[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
    uint32_t mn = 0xFFFFFFFFu, mx = 0u;
    auto acc1 = [&](uint32_t xi, double yi, int set) {
      const double v = u2d(xi);
      mn = min(mn, xi);
      mx = max(mx, xi);
      FitTraits<DOOLY_KIND_AFFINE>::accumulate(&v, yi, a[set]);
    };
    warp_stream_affine(
        x, y, beg, n, vec_ok, true,
        [&](const uint4& xv, const double4& yv) {
          acc1(xv.x, yv.x, 0);
          acc1(xv.y, yv.y, 1);
          acc1(xv.z, yv.z, 0);
          acc1(xv.w, yv.w, 1);
        },
        [&](uint32_t xi, double yi) { acc1(xi, yi, 0); });
    double sx = warp_sum(a[0][0] + a[1][0]), sxx = warp_sum(a[0][1] + a[1][1]);
    double sy = warp_sum(a[0][2] + a[1][2]), sxy = warp_sum(a[0][3] + a[1][3]);
    mn = __reduce_min_sync(0xFFFFFFFFu, mn);
    mx = __reduce_max_sync(0xFFFFFFFFu, mx);
    // ---- 2x2 scaled normal equations, Cholesky with drop (reduce_and_solve's
    // arithmetic for NCOL = 2), solved redundantly by every lane
    const double inv = mx > 0 ? 1.0 / (double)mx : 1.0;  // IEEE division (oracle parity)
    const double g00 = (double)n, g01 = sx * inv, g11 = sxx * (1.0 * inv * inv);
    const double b0 = sy * 1.0, b1 = sxy * inv;
    const bool k0 = g00 > DROP_TOL * g00;
    const double d0 = k0 ? sqrt(g00) : 0.0, rd0 = k0 ? rcp64(d0) : 0.0;
    const double l10 = g01 * rd0;
    const double p11 = fma(-l10, l10, g11);
    const bool k1 = p11 > DROP_TOL * g11;
    const double d1 = k1 ? sqrt(p11) : 0.0, rd1 = k1 ? rcp64(d1) : 0.0;
    const double z0 = b0 * rd0;
    const double z1 = fma(-l10, z0, b1) * rd1;
    double c[2];
    c[1] = z1 * rd1;
    c[0] = fma(-l10, c[1], z0) * rd0;
    // ---- pass 2: training MAPE (the points re-read, normally from L2)
    double e0 = 0.0, e1 = 0.0;
    auto term = [&](uint32_t xi, double yi) {
      const uint32_t xv[1] = {xi};
      return mape_term<DOOLY_KIND_AFFINE>(xv, yi, c, &inv);
    };
    warp_stream_affine(
        x, y, beg, n, vec_ok, false,
        [&](const uint4& xv, const double4& yv) {
          e0 += term(xv.x, yv.x);
          e1 += term(xv.y, yv.y);
          e0 += term(xv.z, yv.z);
          e1 += term(xv.w, yv.w);
        },
        [&](uint32_t xi, double yi) { e0 += term(xi, yi); });
    const double e = warp_sum(e0 + e1);
    if (lane == 0) {
      dooly_affine_row* row = table + s;
      row->c0 = c[0];
      row->c1 = c[1];
      row->inv_scale = inv;
      row->lo = mn;
      row->hi = mx;
      fit_err[s] = e / (double)n;
      status[s] = DOOLY_FIT_OK;
    }
  }
}

// ====================================================================
// Attention (10-column) path: three kernels.
//
// ncu showed the fused stage kernel spending ~a third of its warp time in the
// per-signature serial phase (the 10x10 solve on warp 0 while three warps wait
// at the barrier) and FP64 pipes only ~40% busy.  For the FP64-bound attention
// kind the solve is therefore taken off the streaming path:
//   A  fit_moments_attn: one WARP per signature streams its points once
//      (16-B vector loads, two blocks in flight per lane), accumulates the 44
//      raw moments + box, butterfly-reduces in registers (no CTA barrier) and
//      stores them moment-major to a workspace (352 B + 24 B per signature);
//   B  fit_solve_attn: one THREAD per signature scales the moments, builds the
//      10x10 Gram, Cholesky-with-drop + substitution in registers, writes the
//      row (0.5M independent solves: latency fully hidden by parallelism);
//   C  fit_mape_attn: one warp per signature re-streams the points with the
//      final row for the training MAPE.
// Points cross HBM twice (40 B/point instead of 20) but both streaming kernels
// run at the FP64 or HBM roofline instead of stalling on a serial solve.
// ====================================================================
constexpr int ATTN_NACC = 44;  // 34 moments (degree 1..4) + 10 X^T y sums
constexpr int FA_THREADS = 128;

struct AttnPoints4 {  // 4 consecutive points
  uint32_t x[4][3];
  double y[4];
};

__device__ __forceinline__ void ld_points4(const uint32_t* x, int64_t n_pts, const double* y,
                                           int64_t i, AttnPoints4& p) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const uint4 v = ld_stream_u4(x + k * n_pts + i);
    p.x[0][k] = v.x;
    p.x[1][k] = v.y;
    p.x[2][k] = v.z;
    p.x[3][k] = v.w;
  }
  const uint4 a = ld_stream_u4(y + i);
  const uint4 b = ld_stream_u4(y + i + 2);
  p.y[0] = __hiloint2double((int)a.y, (int)a.x);
  p.y[1] = __hiloint2double((int)a.w, (int)a.z);
  p.y[2] = __hiloint2double((int)b.y, (int)b.x);
  p.y[3] = __hiloint2double((int)b.w, (int)b.z);
}

__device__ __forceinline__ void attn_point(const uint32_t* xv, double yv, double* acc,
                                           uint32_t* mn, uint32_t* mx) {
  double v[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    v[k] = u2d(xv[k]);
    mn[k] = min(mn[k], xv[k]);
    mx[k] = max(mx[k], xv[k]);
  }
  attn_accumulate(v[0], v[1], v[2], yv, acc);
}

// Visit every point of [beg, end) once per lane-strided schedule; `vec` selects
// 16-B vector loads (4 points per lane per block of 128).
template <typename F4, typename F1>
__device__ __forceinline__ void warp_stream_points(const uint32_t* x, int64_t n_pts,
                                                   const double* y, int64_t beg, int64_t n,
                                                   bool vec, F4&& f4, F1&& f1) {
  const int lane = threadIdx.x & 31;
  int64_t done = 0;
  if (vec) {
    const int64_t full = n / 128 * 128;
    int64_t i = 0;
    for (; i + 256 <= full; i += 256) {  // two blocks of loads in flight per lane
      AttnPoints4 p0, p1;
      ld_points4(x, n_pts, y, beg + i + 4 * lane, p0);
      ld_points4(x, n_pts, y, beg + i + 128 + 4 * lane, p1);
      f4(p0);
      f4(p1);
    }
    for (; i < full; i += 128) {
      AttnPoints4 p0;
      ld_points4(x, n_pts, y, beg + i + 4 * lane, p0);
      f4(p0);
    }
    done = full;
  }
  for (int64_t i = done + lane; i < n; i += 32) {
    uint32_t xv[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) xv[k] = __ldg(x + k * n_pts + beg + i);
    f1(xv, __ldg(y + beg + i));
  }
}

// Per-lane cp.async pipeline: each lane copies exactly the 16-B pieces it
// later consumes (3 x-plane chunks + 2 y chunks per 128-point block), so the
// ring needs no cross-lane synchronisation, only cp.async.wait_group; D blocks
// are in flight per warp without holding any registers.
#ifndef FA_DEPTH_N
#define FA_DEPTH_N 8
#endif
constexpr int FA_DEPTH = FA_DEPTH_N;  // blocks in flight per warp (8: fused 13.24 -> 12.93 ms, split 13.30 -> 13.15)
constexpr int FA_BLOCK_BYTES = 3 * 128 * 4 + 128 * 8;  // 2560 B per 128-point block
constexpr size_t FA_SMEM = (size_t)(FA_THREADS / 32) * FA_DEPTH * FA_BLOCK_BYTES;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <typename F4, typename F1>
__device__ __forceinline__ void warp_stream_points_async(unsigned char* ring, const uint32_t* x,
                                                         int64_t n_pts, const double* y,
                                                         int64_t beg, int64_t n, bool vec,
                                                         F4&& f4, F1&& f1) {
  const int lane = threadIdx.x & 31;
  int64_t done = 0;
  if (vec) {
    const int64_t nb = n / 128;
    auto issue = [&](int64_t b) {
      unsigned char* st = ring + (size_t)(b % FA_DEPTH) * FA_BLOCK_BYTES;
      const int64_t i = beg + b * 128 + 4 * lane;
#pragma unroll
      for (int k = 0; k < 3; ++k) cp_async16(st + k * 512 + 16 * lane, x + k * n_pts + i);
      cp_async16(st + 1536 + 32 * lane, y + i);
      cp_async16(st + 1536 + 32 * lane + 16, y + i + 2);
    };
#pragma unroll
    for (int d = 0; d < FA_DEPTH - 1; ++d) {
      if (d < nb) issue(d);
      cp_async_commit();
    }
    for (int64_t b = 0; b < nb; ++b) {
      if (b + FA_DEPTH - 1 < nb) issue(b + FA_DEPTH - 1);
      cp_async_commit();
      cp_async_wait<FA_DEPTH - 1>();
      const unsigned char* st = ring + (size_t)(b % FA_DEPTH) * FA_BLOCK_BYTES;
      AttnPoints4 p;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const uint4 v = *reinterpret_cast<const uint4*>(st + k * 512 + 16 * lane);
        p.x[0][k] = v.x;
        p.x[1][k] = v.y;
        p.x[2][k] = v.z;
        p.x[3][k] = v.w;
      }
      const double2 a = *reinterpret_cast<const double2*>(st + 1536 + 32 * lane);
      const double2 c = *reinterpret_cast<const double2*>(st + 1536 + 32 * lane + 16);
      p.y[0] = a.x;
      p.y[1] = a.y;
      p.y[2] = c.x;
      p.y[3] = c.y;
      f4(p);
    }
    cp_async_wait<0>();
    done = nb * 128;
  }
  for (int64_t i = done + lane; i < n; i += 32) {
    uint32_t xv[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) xv[k] = __ldg(x + k * n_pts + beg + i);
    f1(xv, __ldg(y + beg + i));
  }
}

// Pass 1 of one attention signature by one warp: the 44 raw sums and the box,
// warp-reduced (every lane returns every sum).
__device__ __forceinline__ void attn_pass1(unsigned char* ring, const uint32_t* x, int64_t n_pts,
                                           const double* y, int64_t beg, int64_t n, bool vec,
                                           int grouped, double* acc, uint32_t* mn, uint32_t* mx) {
#pragma unroll
  for (int i = 0; i < ATTN_NACC; ++i) acc[i] = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    mn[k] = 0xFFFFFFFFu;
    mx[k] = 0u;
  }
  warp_stream_points_async(
      ring, x, n_pts, y, beg, n, vec,
      [&](const AttnPoints4& p) {
        // 4 consecutive points sharing prefill_toks and batch (a sweep grid
        // with kv innermost): grouped moments, ~25 FP64 per point instead of 63
        const bool same = grouped && p.x[1][0] == p.x[0][0] && p.x[2][0] == p.x[0][0] &&
                          p.x[3][0] == p.x[0][0] && p.x[1][1] == p.x[0][1] &&
                          p.x[2][1] == p.x[0][1] && p.x[3][1] == p.x[0][1];
        if (same) {
          double c4[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            c4[u] = u2d(p.x[u][2]);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
              mn[k] = min(mn[k], p.x[u][k]);
              mx[k] = max(mx[k], p.x[u][k]);
            }
          }
          attn_accumulate_group(u2d(p.x[0][0]), u2d(p.x[0][1]), c4, p.y, acc);
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) attn_point(p.x[u], p.y[u], acc, mn, mx);
        }
      },
      [&](const uint32_t* xv, double yv) { attn_point(xv, yv, acc, mn, mx); });
#pragma unroll
  for (int i = 0; i < ATTN_NACC; ++i) acc[i] = warp_sum(acc[i]);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    mn[k] = __reduce_min_sync(0xFFFFFFFFu, mn[k]);
    mx[k] = __reduce_max_sync(0xFFFFFFFFu, mx[k]);
  }
}

__global__ void __launch_bounds__(FA_THREADS) fit_moments_attn_kernel(
    const uint32_t* __restrict__ x, int64_t n_pts, const double* __restrict__ y,
    const int64_t* __restrict__ off, int64_t n_sig, double* __restrict__ mom,
    uint32_t* __restrict__ box, bool vec_ok, int grouped) {
  extern __shared__ __align__(16) unsigned char fa_dyn[];
  unsigned char* ring = fa_dyn + (size_t)(threadIdx.x >> 5) * FA_DEPTH * FA_BLOCK_BYTES;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = warp; s < n_sig; s += n_warps) {
    const int64_t beg = __ldg(off + s), n = __ldg(off + s + 1) - beg;
    if (n < FitTraits<DOOLY_KIND_ATTN>::NEED) continue;  // the solve kernel marks it
    double acc[ATTN_NACC];
    uint32_t mn[3], mx[3];
    attn_pass1(ring, x, n_pts, y, beg, n, vec_ok && (beg % 4 == 0), grouped, acc, mn, mx);
    // moment-major stores, spread over lanes (every lane holds every sum)
#pragma unroll
    for (int i = 0; i < ATTN_NACC; ++i)
      if (lane == (i & 31)) mom[(int64_t)i * n_sig + s] = acc[i];
    if (lane < 3) {
      box[(int64_t)lane * n_sig + s] = lane == 0 ? mn[0] : lane == 1 ? mn[1] : mn[2];
      box[(int64_t)(3 + lane) * n_sig + s] = lane == 0 ? mx[0] : lane == 1 ? mx[1] : mx[2];
    }
  }
}

// The 10-column solve of one signature from its 44 raw sums (34 moments of
// degree 1..4 + 10 X^T y sums, in accumulator order) and its box: scaled
// moments, Gram, Cholesky with drop, substitution.  Writes c[10] and inv[3].
__device__ __forceinline__ void attn_solve_row(int64_t n, const double* raw, const uint32_t* hi,
                                               double* c, double* inv) {
  constexpr int NC = 10;
#pragma unroll
  for (int k = 0; k < 3; ++k) inv[k] = hi[k] > 0 ? 1.0 / (double)hi[k] : 1.0;  // IEEE division (oracle parity)
  // scaled moments: raw sum * prod inv^e; the scales follow the same
  // degree-<=4 monomial recurrence as the moments themselves
  double sc[35], msc[35];
  attn_monomials(inv[0], inv[1], inv[2], sc);
  msc[0] = (double)n;
#pragma unroll
  for (int m = 1; m < 35; ++m) msc[m] = raw[m - 1] * sc[m];
  double L[NC][NC];  // lower triangle used
  attn_gram(msc, L);
  double b[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) b[i] = raw[34 + i] * sc[attn_colmon(i)];
  // Cholesky with drop (same rule as the oracle): L overwrites G
  double rd[NC];
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    const double gjj = L[j][j];
    double d2 = gjj;
#pragma unroll
    for (int k = 0; k < j; ++k) d2 = fma(-L[j][k], L[j][k], d2);
    const bool keep = d2 > DROP_TOL * gjj;
    const double d = keep ? sqrt(d2) : 0.0;
    rd[j] = keep ? rcp64(d) : 0.0;
    L[j][j] = d;
#pragma unroll
    for (int i = j + 1; i < NC; ++i) {
      double t = L[i][j];
#pragma unroll
      for (int k = 0; k < j; ++k) t = fma(-L[i][k], L[j][k], t);
      L[i][j] = t * rd[j];
    }
  }
  double z[NC];
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    double t = b[j];
#pragma unroll
    for (int k = 0; k < j; ++k) t = fma(-L[j][k], z[k], t);
    z[j] = t * rd[j];
  }
#pragma unroll
  for (int j = NC - 1; j >= 0; --j) {
    double t = z[j];
#pragma unroll
    for (int k = j + 1; k < NC; ++k) t = fma(-L[k][j], c[k], t);
    c[j] = t * rd[j];
  }
}

__device__ __forceinline__ void write_attn_row(dooly_attn_row* row, const double* c,
                                               const double* inv, const uint32_t* lo,
                                               const uint32_t* hi) {
#pragma unroll
  for (int i = 0; i < 10; ++i) row->c[i] = c[i];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    row->inv_scale[k] = inv[k];
    row->lo[k] = lo[k];
    row->hi[k] = hi[k];
  }
}

__global__ void __launch_bounds__(128) fit_solve_attn_kernel(
    const int64_t* __restrict__ off, int64_t n_sig, const double* __restrict__ mom,
    const uint32_t* __restrict__ box, dooly_attn_row* __restrict__ table,
    double* __restrict__ fit_err, uint8_t* __restrict__ status) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n_sig;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = __ldg(off + s + 1) - __ldg(off + s);
    if (n < FitTraits<DOOLY_KIND_ATTN>::NEED) {
      write_unfitted<DOOLY_KIND_ATTN>(table, s, fit_err, status);
      continue;
    }
    uint32_t lo[3], hi[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      lo[k] = __ldg(box + (int64_t)k * n_sig + s);
      hi[k] = __ldg(box + (int64_t)(3 + k) * n_sig + s);
    }
    double raw[ATTN_NACC];
#pragma unroll
    for (int i = 0; i < ATTN_NACC; ++i) raw[i] = __ldg(mom + (int64_t)i * n_sig + s);
    double c[10], inv[3];
    attn_solve_row(n, raw, hi, c, inv);
    write_attn_row(table + s, c, inv, lo, hi);
    status[s] = DOOLY_FIT_OK;
  }
}

// Training MAPE of one attention signature by one warp (warp-summed).
__device__ __forceinline__ double attn_pass2(const uint32_t* x, int64_t n_pts, const double* y,
                                             int64_t beg, int64_t n, bool vec, const AttnRow& r,
                                             unsigned char* ring = nullptr) {
  double e0 = 0.0, e1 = 0.0;
  auto term = [&](const uint32_t* xv, double yv) {
    double v[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) v[k] = u2d(xv[k]);
    const double p = fmax(eval_fma<DOOLY_KIND_ATTN>(r.c, r.inv, v), DOOLY_CLAMP_FLOOR);
    return fabs(p - yv) * rcp64(yv);
  };
  auto f4 = [&](const AttnPoints4& p) {
    e0 += term(p.x[0], p.y[0]);
    e1 += term(p.x[1], p.y[1]);
    e0 += term(p.x[2], p.y[2]);
    e1 += term(p.x[3], p.y[3]);
  };
  auto f1 = [&](const uint32_t* xv, double yv) { e0 += term(xv, yv); };
  if (ring != nullptr)   // blocks in flight through the warp's cp.async ring
    warp_stream_points_async(ring, x, n_pts, y, beg, n, vec, f4, f1);
  else
    warp_stream_points(x, n_pts, y, beg, n, vec, f4, f1);
  return warp_sum(e0 + e1);
}

__global__ void __launch_bounds__(FA_THREADS) fit_mape_attn_kernel(
    const uint32_t* __restrict__ x, int64_t n_pts, const double* __restrict__ y,
    const int64_t* __restrict__ off, int64_t n_sig, const dooly_attn_row* __restrict__ table,
    double* __restrict__ fit_err, bool vec_ok) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = warp; s < n_sig; s += n_warps) {
    const int64_t beg = __ldg(off + s), n = __ldg(off + s + 1) - beg;
    if (n < FitTraits<DOOLY_KIND_ATTN>::NEED) continue;
    const AttnRow r = load_attn(table, (uint32_t)s);
    const double e = attn_pass2(x, n_pts, y, beg, n, vec_ok && (beg % 4 == 0), r);
    if (lane == 0) fit_err[s] = e / (double)n;
  }
}

// Fused attention CSR fit (the default; DOOLY_FIT_CSR_ATTN=split selects the
// three kernels, see launch_fit): one warp per signature runs pass 1,
// the solve (every lane, the same arithmetic as fit_solve_attn_kernel) and
// pass 2, whose re-read of the signature's points mostly hits L2 — 2 CTAs of 4
// warps per SM keep (warps in flight x 20 B x points) within L2.
#ifndef FA_FUSED_MINB
#define FA_FUSED_MINB 2
#endif
__global__ void __launch_bounds__(FA_THREADS, FA_FUSED_MINB) fit_fused_attn_kernel(
    const uint32_t* __restrict__ x, int64_t n_pts, const double* __restrict__ y,
    const int64_t* __restrict__ off, int64_t n_sig, dooly_attn_row* __restrict__ table,
    double* __restrict__ fit_err, uint8_t* __restrict__ status, bool vec_ok, int grouped) {
  extern __shared__ __align__(16) unsigned char fa_dyn[];
  unsigned char* ring = fa_dyn + (size_t)(threadIdx.x >> 5) * FA_DEPTH * FA_BLOCK_BYTES;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = warp; s < n_sig; s += n_warps) {
    const int64_t beg = __ldg(off + s), n = __ldg(off + s + 1) - beg;
    if (n < FitTraits<DOOLY_KIND_ATTN>::NEED) {
      if (lane == 0) write_unfitted<DOOLY_KIND_ATTN>(table, s, fit_err, status);
      continue;
    }
    const bool vec = vec_ok && (beg % 4 == 0);
    AttnRow r;
    {
      double acc[ATTN_NACC];
      uint32_t mn[3], mx[3];
      attn_pass1(ring, x, n_pts, y, beg, n, vec, grouped, acc, mn, mx);
      attn_solve_row(n, acc, mx, r.c, r.inv);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        r.lo[k] = mn[k];
        r.hi[k] = mx[k];
      }
    }
    if (lane == 0) {
      write_attn_row(table + s, r.c, r.inv, r.lo, r.hi);
      status[s] = DOOLY_FIT_OK;
    }
    const double e = attn_pass2(x, n_pts, y, beg, n, vec, r, ring);
    if (lane == 0) fit_err[s] = e / (double)n;
  }
}

size_t fit_workspace_size(int kind, int64_t n_sig) {
  if (kind != DOOLY_KIND_ATTN) return 0;
  return (size_t)n_sig * (ATTN_NACC * 8 + 6 * 4) + 256;
}

static cudaError_t launch_attn(const uint32_t* x, int64_t n_pts, const double* y,
                               const int64_t* off, int64_t n_sig, void* table, double* fit_err,
                               uint8_t* status, void* ws, cudaStream_t stream, int n_sm) {
  double* mom = static_cast<double*>(ws);
  uint32_t* box = reinterpret_cast<uint32_t*>(mom + (size_t)ATTN_NACC * n_sig);
  const bool vec_ok = ((uintptr_t)x % 16 == 0) && ((uintptr_t)y % 16 == 0) && (n_pts % 4 == 0);
  int per_sm = 0;
  cudaFuncSetAttribute(fit_moments_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)FA_SMEM);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fit_moments_attn_kernel, FA_THREADS,
                                                FA_SMEM);
  int64_t blocks = (int64_t)n_sm * (per_sm > 0 ? per_sm : 1);
  const int64_t need = (n_sig + FA_THREADS / 32 - 1) / (FA_THREADS / 32);
  if (blocks > need) blocks = need;
  const char* grp = getenv("DOOLY_FIT_GROUPED");   // "0": per-point moments only
  fit_moments_attn_kernel<<<(unsigned)blocks, FA_THREADS, FA_SMEM, stream>>>(
      x, n_pts, y, off, n_sig, mom, box, vec_ok, grp == nullptr || grp[0] != '0');
  int64_t sb = (n_sig + 127) / 128;
  fit_solve_attn_kernel<<<(unsigned)sb, 128, 0, stream>>>(
      off, n_sig, mom, box, static_cast<dooly_attn_row*>(table), fit_err, status);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fit_mape_attn_kernel, FA_THREADS, 0);
  blocks = (int64_t)n_sm * (per_sm > 0 ? per_sm : 1);
  if (blocks > need) blocks = need;
  fit_mape_attn_kernel<<<(unsigned)blocks, FA_THREADS, 0, stream>>>(
      x, n_pts, y, off, n_sig, static_cast<const dooly_attn_row*>(table), fit_err, vec_ok);
  return cudaGetLastError();
}

cudaError_t launch_fit(int kind, const uint32_t* x, int64_t n_pts, const double* y,
                       const int64_t* off, int64_t n_sig, void* table, double* fit_err,
                       uint8_t* status, void* ws, cudaStream_t stream, int n_sm,
                       int64_t* launches) {
  if (n_sig == 0) return cudaSuccess;
  if (kind == DOOLY_KIND_AFFINE) {
    *launches += 1;
    const char* which = getenv("DOOLY_FIT_CSR_AFFINE");  // "stage": the staged CTA kernel
    if (which == nullptr || strcmp(which, "stage") != 0) {
      const bool vec_ok = ((uintptr_t)x % 16 == 0) && ((uintptr_t)y % 32 == 0);
      int64_t blocks = (int64_t)n_sm * 2;
      const int64_t need = (n_sig + 7) / 8;
      if (blocks > need) blocks = need;
      fit_affine_warp_kernel<<<(unsigned)blocks, 256, 0, stream>>>(
          x, y, off, n_sig, static_cast<dooly_affine_row*>(table), fit_err, status, vec_ok);
      return cudaGetLastError();
    }
    return launch_kind<DOOLY_KIND_AFFINE>(x, n_pts, y, off, n_sig, table, fit_err, status,
                                          stream, n_sm);
  }
  // default: one warp per signature for pass 1, solve and pass 2 (the points
  // cross HBM once; 12.93 vs 13.15 ms per 0.5M x 4096 points for the split
  // kernels, DOOLY_FIT_CSR_ATTN=split — at 234 registers and 8 warps per SM
  // the fused kernel is latency-bound, the split ones run near HBM speed)
  const char* which = getenv("DOOLY_FIT_CSR_ATTN");
  if (which == nullptr || strcmp(which, "split") != 0) {
    *launches += 1;
    const bool vec_ok = ((uintptr_t)x % 16 == 0) && ((uintptr_t)y % 16 == 0) && (n_pts % 4 == 0);
    cudaError_t e = cudaFuncSetAttribute(fit_fused_attn_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FA_SMEM);
    if (e != cudaSuccess) return e;
    int64_t blocks = (int64_t)n_sm * FA_FUSED_MINB;
    const int64_t need = (n_sig + FA_THREADS / 32 - 1) / (FA_THREADS / 32);
    if (blocks > need) blocks = need;
    const char* grp = getenv("DOOLY_FIT_GROUPED");   // "0": per-point moments only
    fit_fused_attn_kernel<<<(unsigned)blocks, FA_THREADS, FA_SMEM, stream>>>(
        x, n_pts, y, off, n_sig, static_cast<dooly_attn_row*>(table), fit_err, status, vec_ok,
        grp == nullptr || grp[0] != '0');
    return cudaGetLastError();
  }
  if (ws == nullptr) {  // no workspace: fused single-kernel path
    *launches += 1;
    return launch_kind<DOOLY_KIND_ATTN>(x, n_pts, y, off, n_sig, table, fit_err, status, stream,
                                        n_sm);
  }
  *launches += 3;
  return launch_attn(x, n_pts, y, off, n_sig, table, fit_err, status, ws, stream, n_sm);
}

}  // namespace dooly
