// K2 — batched per-signature least-squares fit (replaces fit).
//
// Data path (B200): a persistent kernel, one 256-thread CTA per SM.  Thread 0
// streams whole signatures (feature planes + latencies) from HBM into a ring
// of shared-memory stages with the bulk-copy (1-D TMA) engine
// (`cp.async.bulk` + mbarrier complete_tx), STAGES-1 signatures ahead of the
// one being computed, so HBM streaming overlaps the FP64 work and the serial
// reduce/solve phases.  Both passes over a signature then read shared memory:
// every point is fetched from HBM exactly once.  Signatures larger than a
// stage fall back to a direct global-memory path (same arithmetic).
//
// Per signature:
//   pass 1  raw power moments sum x^a y^b z^c (a+b+c <= 4: 35 for attention,
//           3 for affine), X^T y for the design monomials, and the training
//           box.  All terms are non-negative so the raw sums are well
//           conditioned; the scaled Gram G[i][j] = M[e_i+e_j] * prod inv^e is
//           formed once per signature (35 moments replace 55 Gram products
//           per point).
//   reduce  warp shuffles -> shared memory -> 8-way column sums.
//   solve   warp 0 factors G with a right-looking Cholesky, one lane per row;
//           columns whose pivot falls to <= DROP_TOL x their diagonal are
//           dropped (rank-deficient designs), then forward/back
//           substitution by shuffles.
//   pass 2  training MAPE (fit_error) of the clamped predictor.
// FP64 throughout; no tensor cores (B200's FP64 tensor peak equals the FP64
// vector peak and lower precisions cannot meet the 1e-9 contract).
#include "attn_moments.cuh"
#include "common.cuh"

namespace dooly {

constexpr double DROP_TOL = 1e-9;
constexpr int FIT_THREADS = 256;
constexpr int FIT_WARPS = FIT_THREADS / 32;
constexpr int FIT_CAP = 4096;  // points per shared-memory stage

template <int KIND>
struct FitTraits;

template <>
struct FitTraits<DOOLY_KIND_AFFINE> {
  static constexpr int P = 1;     // features
  static constexpr int NCOL = 2;  // design columns [1, f]
  static constexpr int NMOM = 3;  // 1, x, x^2
  static constexpr int NEED = 4;  // max(4, NCOL + 1)   (App. A.8)
  static constexpr int STAGES = 3;
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
  static constexpr int STAGES = 2;
  __device__ static __forceinline__ void monomials(const double* v, double* m) {
    attn_monomials(v[0], v[1], v[2], m);
  }
  // dynamic-index lookups (Gram assembly, once per signature) use __constant__ tables
  __device__ static __forceinline__ int colmon(int i) { return kAttnColmon[i]; }
  __device__ static __forceinline__ int gidx(int i, int j) { return kAttnGidx[i][j]; }
  __device__ static __forceinline__ int exp(int m, int k) { return kAttnExp[m][k]; }
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

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}

template <int KIND>
__device__ __forceinline__ double eval_row(const double* c, const double* inv,
                                           const uint32_t* xs) {
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
  static constexpr int P = FitTraits<KIND>::P, NCOL = FitTraits<KIND>::NCOL,
                       NACC = FitTraits<KIND>::NMOM - 1 + FitTraits<KIND>::NCOL;
  double part[FIT_WARPS][NACC];
  uint32_t mn[FIT_WARPS][P], mx[FIT_WARPS][P];
  double mom[NACC];
  double G[NCOL][NCOL + 1];
  double b[NCOL];
  double coef[NCOL];
  double inv[P];
  uint32_t lo[P], hi[P];
  double err[FIT_WARPS];
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

// Fit one signature with n >= NEED points; all threads of the CTA participate.
template <int KIND, typename Pts>
__device__ void fit_one(const Pts& pts, int64_t n, int64_t s, FitScratch<KIND>& sh, void* table,
                        double* fit_err, uint8_t* status) {
  using T = FitTraits<KIND>;
  constexpr int P = T::P, NCOL = T::NCOL, NMOM = T::NMOM;
  constexpr int NACC = (NMOM - 1) + NCOL;
  constexpr int UNR = 4;
  constexpr int kAffineColmon[2] = {0, 1};
  constexpr int kAttnColmonStatic[10] = DOOLY_ATTN_COLMON;
  const int* kColmon = KIND == DOOLY_KIND_AFFINE ? kAffineColmon : kAttnColmonStatic;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

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
  for (int64_t i0 = tid; i0 < n; i0 += FIT_THREADS * UNR) {
    uint32_t xv[UNR][P];
    double yv[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t i = i0 + u * FIT_THREADS;
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
      if (i0 + u * FIT_THREADS >= n) break;
      double mon[NMOM];
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
      for (int i = 0; i < NCOL; ++i)
        acc[NMOM - 1 + i] = fma(yv[u], mon[kColmon[i]], acc[NMOM - 1 + i]);
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
    for (int i = 0; i < NACC; ++i) sh.part[wid][i] = acc[i];
#pragma unroll
    for (int k = 0; k < P; ++k) {
      sh.mn[wid][k] = mn[k];
      sh.mx[wid][k] = mx[k];
    }
  }
  __syncthreads();
  if (tid < NACC) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < FIT_WARPS; ++w) t += sh.part[w][tid];
    sh.mom[tid] = t;
  } else if (tid >= 64 && tid < 64 + P) {
    const int k = tid - 64;
    uint32_t a = 0xFFFFFFFFu, b = 0u;
#pragma unroll
    for (int w = 0; w < FIT_WARPS; ++w) {
      a = min(a, sh.mn[w][k]);
      b = max(b, sh.mx[w][k]);
    }
    sh.lo[k] = a;
    sh.hi[k] = b;
    sh.inv[k] = b > 0 ? 1.0 / (double)b : 1.0;  // IEEE division: bit-identical to the oracle
  }
  __syncthreads();
  // ---------------- scaled Gram / rhs (one entry per thread)
  if (tid < NCOL * NCOL + NCOL) {
    const int i = tid < NCOL * NCOL ? tid / NCOL : tid - NCOL * NCOL;
    const int j = tid < NCOL * NCOL ? tid % NCOL : -1;
    const int m = j >= 0 ? T::gidx(i, j) : T::colmon(i);
    double scl = 1.0;
    for (int k = 0; k < P; ++k)
      for (int r = 0; r < T::exp(m, k); ++r) scl *= sh.inv[k];
    if (j >= 0)
      sh.G[i][j] = (m == 0 ? (double)n : sh.mom[m - 1]) * scl;
    else
      sh.b[i] = sh.mom[NMOM - 1 + i] * scl;
  }
  __syncthreads();
  // ---------------- solve: warp 0, lane i owns row i
  if (wid == 0) {
    const int r = lane < NCOL ? lane : 0;
    double g[NCOL];
#pragma unroll
    for (int k = 0; k < NCOL; ++k) g[k] = sh.G[r][k];
    const double diag = sh.G[r][r];
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
    double t = lane < NCOL ? sh.b[lane] : 0.0, z = 0.0;
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
  for (int64_t i0 = tid; i0 < n; i0 += FIT_THREADS * UNR) {
    uint32_t xv[UNR][P];
    double yv[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t i = i0 + u * FIT_THREADS;
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
      if (i0 + u * FIT_THREADS >= n) break;
      bool cl;
      const double p = clamp_floor(eval_row<KIND>(coef, inv, xv[u]), cl);
      err += fabs(p - yv[u]) * rcp64(yv[u]);
    }
  }
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
  __syncthreads();  // shared scratch reused by the next signature
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

// Issue the bulk copies of signature s into stage memory; returns nothing, the
// tail elements beyond the aligned window are loaded by the consumers.
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
__global__ void __launch_bounds__(FIT_THREADS, 1) fit_bulk_kernel(
    const uint32_t* __restrict__ x, int64_t n_pts, const double* __restrict__ y,
    const int64_t* __restrict__ off, int64_t n_sig, void* __restrict__ table,
    double* __restrict__ fit_err, uint8_t* __restrict__ status, bool bulk_ok) {
  using T = FitTraits<KIND>;
  using S = Stage<KIND>;
  constexpr int NST = T::STAGES;
  extern __shared__ __align__(128) unsigned char dyn[];
  __shared__ __align__(8) uint64_t bars[NST];
  __shared__ FitScratch<KIND> sh;
  const int tid = threadIdx.x;

  // signatures of this CTA: s_k = blockIdx.x + k * gridDim.x
  auto sig_of = [&](int64_t k) { return (int64_t)blockIdx.x + k * (int64_t)gridDim.x; };
  auto stageable = [&](int64_t s) {
    const int64_t n = off[s + 1] - off[s];
    return bulk_ok && n >= T::NEED && n <= FIT_CAP;
  };
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
  uint32_t phase_bits = 0;  // per-stage parity
  for (int64_t k = 0;; ++k) {
    const int64_t s = sig_of(k);
    if (s >= n_sig) break;
    // keep STAGES-1 signatures in flight: refill the stage freed at the end of k-1
    if (tid == 0) {
      const int64_t kn = k + NST - 1;
      const int64_t sn = sig_of(kn);
      if (sn < n_sig && stageable(sn)) {
        const int st = (int)(kn % NST);
        issue_stage<KIND>(dyn + (size_t)st * S::STRIDE, &bars[st], x, n_pts, y, off[sn],
                          off[sn + 1]);
      }
    }
    const int64_t beg = off[s], end = off[s + 1], n = end - beg;
    if (n < T::NEED) {
      if (tid == 0) write_unfitted<KIND>(table, s, fit_err, status);
      continue;  // no stage was used (stageable() is false)
    }
    if (!stageable(s)) {  // oversized / unaligned inputs: stream straight from global memory
      GlobalPoints<T::P> gp{x, n_pts, y, beg};
      fit_one<KIND>(gp, n, s, sh, table, fit_err, status);
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
    fit_one<KIND>(sp, n, s, sh, table, fit_err, status);  // ends with __syncthreads
  }
}

template <int KIND>
static cudaError_t launch_kind(const uint32_t* x, int64_t n_pts, const double* y,
                               const int64_t* off, int64_t n_sig, void* table, double* fit_err,
                               uint8_t* status, cudaStream_t stream, int n_sm) {
  const size_t smem = (size_t)FitTraits<KIND>::STAGES * Stage<KIND>::STRIDE;
  cudaError_t e = cudaFuncSetAttribute(fit_bulk_kernel<KIND>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // 1-D TMA needs 16-B aligned sources: plane bases and the y array
  const bool bulk_ok = ((uintptr_t)x % 16 == 0) && ((uintptr_t)y % 16 == 0) &&
                       (FitTraits<KIND>::P == 1 || n_pts % 4 == 0);
  int64_t blocks = n_sm;
  if (blocks > n_sig) blocks = n_sig;
  fit_bulk_kernel<KIND><<<(unsigned)blocks, FIT_THREADS, smem, stream>>>(
      x, n_pts, y, off, n_sig, table, fit_err, status, bulk_ok);
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
