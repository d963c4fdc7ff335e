// K2 — batched per-signature least-squares fit (replaces fit).
//
// One 256-thread CTA per signature (persistent grid-stride over signatures):
//   pass 1  every thread strides over the signature's points (coalesced 4-B
//           feature loads, 8-B latency loads, 4-deep unrolled so 16 points of
//           loads are in flight per thread) and accumulates RAW power moments
//           sum x^a y^b z^c (a+b+c <= 4; 35 for attention, 3 for affine) and
//           sum y*m for the design monomials, plus the training box.
//           All terms are non-negative, so raw-moment sums are well
//           conditioned; the scaled Gram G[i][j] = M[e_i+e_j] * prod inv^e
//           is formed once per signature (35 moments replace 55 Gram
//           products per point: ~75 FP64 instructions per point instead of
//           ~130).
//   reduce  warp shuffles -> shared memory -> 8-way column sums.
//   solve   warp 0 factors G with a right-looking Cholesky, one lane per row,
//           columns whose pivot falls below DROP_TOL * original diagonal are
//           dropped (rank-deficient designs), then forward/back
//           substitution by shuffles.
//   pass 2  training MAPE (fit_error): the points are re-read — they were
//           streamed microseconds ago by this CTA and are L2-resident (126 MB
//           L2 >> CTAs-in-flight x 80 KB) — so DRAM traffic stays ~1x.
// FP64 throughout; no tensor cores (FP64 tensor peak == FP64 vector peak on
// B200 and lower precisions cannot meet the 1e-9 contract).
#include "common.cuh"
#include "attn_moments.cuh"

namespace dooly {

constexpr double DROP_TOL = 1e-9;
constexpr int FIT_THREADS = 256;
constexpr int FIT_WARPS = FIT_THREADS / 32;

template <int KIND>
struct FitTraits;

template <>
struct FitTraits<DOOLY_KIND_AFFINE> {
  static constexpr int P = 1;     // features
  static constexpr int NCOL = 2;  // design columns [1, f]
  static constexpr int NMOM = 3;  // 1, x, x^2
  static constexpr int NEED = 4;  // max(4, NCOL + 1)   (App. A.8)
  __device__ static __forceinline__ void monomials(const double* v, double* m) {
    m[0] = 1.0;
    m[1] = v[0];
    m[2] = v[0] * v[0];
  }
  __device__ static __forceinline__ int colmon(int i) { return i; }
  __device__ static __forceinline__ int gidx(int i, int j) { return i + j; }
  __device__ static __forceinline__ int exp(int m, int) { return m; }
};

template <>
struct FitTraits<DOOLY_KIND_ATTN> {
  static constexpr int P = 3;
  static constexpr int NCOL = 10;
  static constexpr int NMOM = 35;
  static constexpr int NEED = 11;
  __device__ static __forceinline__ void monomials(const double* v, double* m) {
    attn_monomials(v[0], v[1], v[2], m);
  }
  // dynamic-index lookups (Gram assembly, once per signature) use __constant__ tables
  __device__ static __forceinline__ int colmon(int i) { return kAttnColmon[i]; }
  __device__ static __forceinline__ int gidx(int i, int j) { return kAttnGidx[i][j]; }
  __device__ static __forceinline__ int exp(int m, int k) { return kAttnExp[m][k]; }
};

__device__ __forceinline__ double rcp64(double y) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y));
  double e = fma(-y, r, 1.0);
  r = fma(r, e, r);
  e = fma(-y, r, 1.0);
  return fma(r, e, r);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}

template <int KIND>
__device__ __forceinline__ double eval_row(const double* c, const double* inv, const uint32_t* xs) {
  if constexpr (KIND == DOOLY_KIND_AFFINE) {
    AffineRow r;
    r.c0 = c[0];
    r.c1 = c[1];
    r.inv = inv[0];
    return eval_affine(r, xs[0]);
  } else {
    AttnRow r;
#pragma unroll
    for (int i = 0; i < 10; ++i) r.c[i] = c[i];
#pragma unroll
    for (int k = 0; k < 3; ++k) r.inv[k] = inv[k];
    return eval_attn(r, xs[0], xs[1], xs[2]);
  }
}

template <int KIND>
__global__ void __launch_bounds__(FIT_THREADS, 2) fit_kernel(
    const uint32_t* __restrict__ x, int64_t n_pts, const double* __restrict__ y,
    const int64_t* __restrict__ off, int64_t n_sig, void* __restrict__ table,
    double* __restrict__ fit_err, uint8_t* __restrict__ status) {
  using T = FitTraits<KIND>;
  constexpr int P = T::P, NCOL = T::NCOL, NMOM = T::NMOM;
  constexpr int NACC = (NMOM - 1) + NCOL;  // moments except n, plus X^T y
  constexpr int UNR = 4;
  constexpr int kAffineColmon[2] = {0, 1};
  constexpr int kAttnColmonStatic[10] = DOOLY_ATTN_COLMON;
  const int* kColmon = KIND == DOOLY_KIND_AFFINE ? kAffineColmon : kAttnColmonStatic;

  __shared__ double s_part[FIT_WARPS][NACC];
  __shared__ uint32_t s_min[FIT_WARPS][P], s_max[FIT_WARPS][P];
  __shared__ double s_mom[NACC];
  __shared__ double s_G[NCOL][NCOL + 1];
  __shared__ double s_b[NCOL];
  __shared__ double s_coef[NCOL];
  __shared__ double s_inv[P];
  __shared__ uint32_t s_lo[P], s_hi[P];
  __shared__ double s_err[FIT_WARPS];

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

  for (int64_t s = blockIdx.x; s < n_sig; s += gridDim.x) {
    const int64_t beg = off[s], end = off[s + 1], n = end - beg;
    if (n < T::NEED) {  // uniform branch: InsufficientData
      if (tid == 0) {
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
      continue;
    }

    // ---------------- pass 1: raw moments + box
    double acc[NACC];
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = 0.0;
    uint32_t mn[P], mx[P];
#pragma unroll
    for (int k = 0; k < P; ++k) {
      mn[k] = 0xFFFFFFFFu;
      mx[k] = 0u;
    }
    for (int64_t j0 = beg + tid; j0 < end; j0 += FIT_THREADS * UNR) {
      uint32_t xv[UNR][P];
      double yv[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int64_t j = j0 + u * FIT_THREADS;
        const bool in = j < end;
#pragma unroll
        for (int k = 0; k < P; ++k) xv[u][k] = in ? __ldg(x + k * n_pts + j) : 0u;
        yv[u] = in ? __ldg(y + j) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        if (j0 + u * FIT_THREADS >= end) break;
        double mon[NMOM];
        mon[0] = 1.0;
        double v[P];
#pragma unroll
        for (int k = 0; k < P; ++k) {
          v[k] = (double)xv[u][k];
          mn[k] = min(mn[k], xv[u][k]);
          mx[k] = max(mx[k], xv[u][k]);
        }
        T::monomials(v, mon);
#pragma unroll
        for (int m = 1; m < NMOM; ++m) acc[m - 1] += mon[m];
#pragma unroll
        for (int i = 0; i < NCOL; ++i) acc[NMOM - 1 + i] = fma(yv[u], mon[kColmon[i]], acc[NMOM - 1 + i]);
      }
    }
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = warp_sum(acc[i]);
#pragma unroll
    for (int k = 0; k < P; ++k) {
      mn[k] = __reduce_min_sync(0xFFFFFFFFu, mn[k]);
      mx[k] = __reduce_max_sync(0xFFFFFFFFu, mx[k]);
    }
    if (lane == 0) {
#pragma unroll
      for (int i = 0; i < NACC; ++i) s_part[wid][i] = acc[i];
#pragma unroll
      for (int k = 0; k < P; ++k) {
        s_min[wid][k] = mn[k];
        s_max[wid][k] = mx[k];
      }
    }
    __syncthreads();
    if (tid < NACC) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < FIT_WARPS; ++w) t += s_part[w][tid];
      s_mom[tid] = t;
    } else if (tid >= 64 && tid < 64 + P) {
      const int k = tid - 64;
      uint32_t a = 0xFFFFFFFFu, b = 0u;
#pragma unroll
      for (int w = 0; w < FIT_WARPS; ++w) {
        a = min(a, s_min[w][k]);
        b = max(b, s_max[w][k]);
      }
      s_lo[k] = a;
      s_hi[k] = b;
      s_inv[k] = b > 0 ? 1.0 / (double)b : 1.0;  // IEEE division: bit-identical to oracle
    }
    __syncthreads();
    // ---------------- scaled Gram / rhs (one entry per thread)
    if (tid < NCOL * NCOL + NCOL) {
      const int i = tid < NCOL * NCOL ? tid / NCOL : tid - NCOL * NCOL;
      const int j = tid < NCOL * NCOL ? tid % NCOL : -1;
      const int m = j >= 0 ? T::gidx(i, j) : T::colmon(i);
      double scl = 1.0;
      for (int k = 0; k < P; ++k)
        for (int r = 0; r < T::exp(m, k); ++r) scl *= s_inv[k];
      if (j >= 0) {
        const double raw = m == 0 ? (double)n : s_mom[m - 1];
        s_G[i][j] = raw * scl;
      } else {
        s_b[i] = s_mom[NMOM - 1 + i] * scl;
      }
    }
    __syncthreads();
    // ---------------- solve: warp 0, lane i owns row i
    if (wid == 0) {
      const int r = lane < NCOL ? lane : 0;
      double g[NCOL];
#pragma unroll
      for (int k = 0; k < NCOL; ++k) g[k] = s_G[r][k];
      const double diag = s_G[r][r];
      uint32_t keep = 0;
#pragma unroll
      for (int j = 0; j < NCOL; ++j) {
        const double piv = __shfl_sync(0xFFFFFFFFu, g[j], j);
        const double dj = __shfl_sync(0xFFFFFFFFu, diag, j);
        const bool kj = piv > DROP_TOL * dj;
        keep |= (uint32_t)kj << j;
        const double d = kj ? sqrt(piv) : 0.0;
        double lij = (kj && lane > j) ? g[j] / d : 0.0;
        if (lane == j) lij = d;
        if (lane >= j) g[j] = lij;
#pragma unroll
        for (int k = j + 1; k < NCOL; ++k) {
          const double lkj = __shfl_sync(0xFFFFFFFFu, lij, k);
          g[k] -= lij * lkj;
        }
      }
      // forward: L z = b
      double t = lane < NCOL ? s_b[lane] : 0.0, z = 0.0;
#pragma unroll
      for (int j = 0; j < NCOL; ++j) {
        const bool kj = (keep >> j) & 1u;
        const double zl = (kj && lane == j) ? t / g[j] : 0.0;
        const double zj = __shfl_sync(0xFFFFFFFFu, zl, j);
        if (lane > j) t -= g[j] * zj;
        if (lane == j) z = zj;
      }
      // backward: L^T c = z
      double u = z, c = 0.0;
#pragma unroll
      for (int j = NCOL - 1; j >= 0; --j) {
        const bool kj = (keep >> j) & 1u;
        const double cl = (kj && lane == j) ? u / g[j] : 0.0;
        const double cj = __shfl_sync(0xFFFFFFFFu, cl, j);
        if (lane == j) c = cj;
#pragma unroll
        for (int m = 0; m < j; ++m) {
          const double ljm = __shfl_sync(0xFFFFFFFFu, g[m], j);  // L[j][m] from lane j
          if (lane == m) u -= ljm * cj;
        }
      }
      if (lane < NCOL) s_coef[lane] = c;
    }
    __syncthreads();
    // ---------------- pass 2: training MAPE with the final (clamped) predictor
    double coef[NCOL], inv[P];
#pragma unroll
    for (int i = 0; i < NCOL; ++i) coef[i] = s_coef[i];
#pragma unroll
    for (int k = 0; k < P; ++k) inv[k] = s_inv[k];
    double err = 0.0;
    for (int64_t j0 = beg + tid; j0 < end; j0 += FIT_THREADS * UNR) {
      uint32_t xv[UNR][P];
      double yv[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int64_t j = j0 + u * FIT_THREADS;
        const bool in = j < end;
#pragma unroll
        for (int k = 0; k < P; ++k) xv[u][k] = in ? __ldg(x + k * n_pts + j) : 0u;
        yv[u] = in ? __ldg(y + j) : 1.0;
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        if (j0 + u * FIT_THREADS >= end) break;
        bool cl;
        const double p = clamp_floor(eval_row<KIND>(coef, inv, xv[u]), cl);
        err += fabs(p - yv[u]) * rcp64(yv[u]);
      }
    }
    err = warp_sum(err);
    if (lane == 0) s_err[wid] = err;
    __syncthreads();
    if (tid == 0) {
      double e = 0.0;
#pragma unroll
      for (int w = 0; w < FIT_WARPS; ++w) e += s_err[w];
      fit_err[s] = e / (double)n;
      status[s] = DOOLY_FIT_OK;
      if constexpr (KIND == DOOLY_KIND_AFFINE) {
        dooly_affine_row* row = static_cast<dooly_affine_row*>(table) + s;
        row->c0 = coef[0];
        row->c1 = coef[1];
        row->inv_scale = inv[0];
        row->lo = s_lo[0];
        row->hi = s_hi[0];
      } else {
        dooly_attn_row* row = static_cast<dooly_attn_row*>(table) + s;
        for (int i = 0; i < 10; ++i) row->c[i] = coef[i];
        for (int k = 0; k < 3; ++k) {
          row->inv_scale[k] = inv[k];
          row->lo[k] = s_lo[k];
          row->hi[k] = s_hi[k];
        }
      }
    }
    __syncthreads();  // shared scratch reused by the next signature
  }
}

cudaError_t launch_fit(int kind, const uint32_t* x, int64_t n_pts, const double* y,
                       const int64_t* off, int64_t n_sig, void* table, double* fit_err,
                       uint8_t* status, cudaStream_t stream, int n_sm) {
  if (n_sig == 0) return cudaSuccess;
  int per_sm = 0;
  if (kind == DOOLY_KIND_AFFINE) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fit_kernel<DOOLY_KIND_AFFINE>,
                                                  FIT_THREADS, 0);
    int64_t blocks = (int64_t)n_sm * (per_sm > 0 ? per_sm : 1);
    if (blocks > n_sig) blocks = n_sig;
    fit_kernel<DOOLY_KIND_AFFINE><<<(unsigned)blocks, FIT_THREADS, 0, stream>>>(
        x, n_pts, y, off, n_sig, table, fit_err, status);
  } else {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fit_kernel<DOOLY_KIND_ATTN>,
                                                  FIT_THREADS, 0);
    int64_t blocks = (int64_t)n_sm * (per_sm > 0 ? per_sm : 1);
    if (blocks > n_sig) blocks = n_sig;
    fit_kernel<DOOLY_KIND_ATTN><<<(unsigned)blocks, FIT_THREADS, 0, stream>>>(
        x, n_pts, y, off, n_sig, table, fit_err, status);
  }
  return cudaGetLastError();
}

}  // namespace dooly
