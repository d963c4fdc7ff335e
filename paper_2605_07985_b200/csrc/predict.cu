// K3 — batched latency prediction (replaces predict).
//
// Gather/evaluate/stream kernel.  Per query the algorithmic HBM traffic is
// sig (4 B) + features (4 B per u32 plane) + latency out (8 B) + 2 flag bits;
// the regressor row (32 B affine / 128 B attention) is an L2-resident gather.
//
// Measured on B200 (profiles/): the first version, with 16-B vector accesses,
// was bound by L1TEX wavefronts of the divergent row gathers (one wavefront
// per distinct line per LDG: 2 per affine row, 8 per attention row), not by
// HBM.  This version is built around sm_100's 256-bit global accesses:
//   * every row sector is fetched with one LDG.256 (affine: 1 per query,
//     attention: 4 per query) tagged L2::evict_last so the table stays in L2;
//   * each lane owns 8 consecutive queries: sig and every feature plane are one
//     LDG.256 each and the 8 latencies are two STG.256, all L2::evict_first
//     (the 10^9-query stream must not evict the table);
//   * flag bits are assembled with warp shuffles (lanes 4w..4w+3 own word w of
//     each 256-query tile) — no atomics, no byte stores;
//   * grid = resident CTAs x 148 SMs, grid-stride over 256-query tiles.
// The evaluation itself (common.cuh) is the bit-exact parity contract.
#include "common.cuh"

namespace dooly {

template <int KIND>
struct Planes {
  static constexpr int P = KIND == DOOLY_KIND_ATTN ? 3 : 1;
};

struct U8 {
  uint32_t v[8];
};

__device__ __forceinline__ U8 ld_stream_256(const uint32_t* p) {
  U8 r;
  asm("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]),
        "=r"(r.v[6]), "=r"(r.v[7])
      : "l"(p));
  return r;
}

__device__ __forceinline__ void ld_row_256(const void* p, double& a, double& b, double& c,
                                           double& d) {
  asm("ld.global.nc.L1::no_allocate.L2::evict_last.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
               : "l"(p));
}

__device__ __forceinline__ void st_stream_256(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.L1::no_allocate.L2::evict_first.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p),
               "d"(a), "d"(b), "d"(c), "d"(d)
               : "memory");
}

__device__ __forceinline__ uint32_t lo32(double d) { return (uint32_t)__double_as_longlong(d); }
__device__ __forceinline__ uint32_t hi32(double d) {
  return (uint32_t)(__double_as_longlong(d) >> 32);
}

// Gather one row with 256-bit loads.
__device__ __forceinline__ AffineRow gather_affine(const dooly_affine_row* t, uint32_t s) {
  AffineRow r;
  double box;
  ld_row_256(t + s, r.c0, r.c1, r.inv, box);
  r.lo = lo32(box);
  r.hi = hi32(box);
  return r;
}

__device__ __forceinline__ AttnRow gather_attn(const dooly_attn_row* t, uint32_t s) {
  const double* p = reinterpret_cast<const double*>(t + s);
  AttnRow r;
  double w6, w7a, w7b;
  ld_row_256(p, r.c[0], r.c[1], r.c[2], r.c[3]);
  ld_row_256(p + 4, r.c[4], r.c[5], r.c[6], r.c[7]);
  ld_row_256(p + 8, r.c[8], r.c[9], r.inv[0], r.inv[1]);
  ld_row_256(p + 12, r.inv[2], w6, w7a, w7b);
  r.lo[0] = lo32(w6);
  r.lo[1] = hi32(w6);
  r.lo[2] = lo32(w7a);
  r.hi[0] = hi32(w7a);
  r.hi[1] = lo32(w7b);
  r.hi[2] = hi32(w7b);
  return r;
}

template <int KIND>
__device__ __forceinline__ double eval_query(const void* table, int64_t n_sig, uint32_t s,
                                             const uint32_t* xs, bool& extrap, bool& clamped,
                                             bool& bad) {
  extrap = clamped = false;
  if (s >= (uint64_t)n_sig) {
    bad = true;
    return nan64();
  }
  if constexpr (KIND == DOOLY_KIND_AFFINE) {
    const AffineRow r = gather_affine(static_cast<const dooly_affine_row*>(table), s);
    if (!affine_valid(r)) {
      bad = true;
      return nan64();
    }
    extrap = xs[0] < r.lo || xs[0] > r.hi;
    return clamp_floor(eval_affine(r, xs[0]), clamped);
  } else {
    const AttnRow r = gather_attn(static_cast<const dooly_attn_row*>(table), s);
    if (!attn_valid(r)) {
      bad = true;
      return nan64();
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) extrap |= xs[k] < r.lo[k] || xs[k] > r.hi[k];
    return clamp_floor(eval_attn(r, xs[0], xs[1], xs[2]), clamped);
  }
}

// Vector path: 256-query tiles, sig / planes / out 32-B aligned, n_q % 8 == 0
// when there is more than one plane.
template <int KIND>
__global__ void __launch_bounds__(256) predict_vec_kernel(
    const void* __restrict__ table, int64_t n_sig, const uint32_t* __restrict__ sig,
    const uint32_t* __restrict__ x, int64_t n_q, double* __restrict__ out,
    uint32_t* __restrict__ flags, int64_t* __restrict__ err_first) {
  constexpr int P = Planes<KIND>::P;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n_tiles = (n_q + 255) >> 8;
  const int64_t n_words = (n_q + 31) >> 5;
  int64_t bad_min = INT64_MAX;

  for (int64_t tile = warp; tile < n_tiles; tile += n_warps) {
    const int64_t q = (tile << 8) + lane * 8;
    U8 sv, xv[P];
    const bool full = q + 8 <= n_q;
    if (full) {
      sv = ld_stream_256(sig + q);
#pragma unroll
      for (int p = 0; p < P; ++p) xv[p] = ld_stream_256(x + p * n_q + q);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const bool in = q + j < n_q;
        sv.v[j] = in ? sig[q + j] : 0u;
#pragma unroll
        for (int p = 0; p < P; ++p) xv[p].v[j] = in ? x[p * n_q + q + j] : 0u;
      }
    }
    double r[8];
    uint32_t ebits = 0, cbits = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t xs[P];
#pragma unroll
      for (int p = 0; p < P; ++p) xs[p] = xv[p].v[j];
      bool e = false, c = false, bad = false;
      if (q + j < n_q) {
        r[j] = eval_query<KIND>(table, n_sig, sv.v[j], xs, e, c, bad);
        if (bad && q + j < bad_min) bad_min = q + j;
      } else {
        r[j] = 0.0;
      }
      ebits |= (uint32_t)e << j;
      cbits |= (uint32_t)c << j;
    }
    if (full) {
      st_stream_256(out + q, r[0], r[1], r[2], r[3]);
      st_stream_256(out + q + 4, r[4], r[5], r[6], r[7]);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (q + j < n_q) out[q + j] = r[j];
    }
    if (flags != nullptr) {
      const int sh = 8 * (lane & 3);
      uint32_t we = ebits << sh, wc = cbits << sh;
      we |= __shfl_xor_sync(0xFFFFFFFFu, we, 1);
      wc |= __shfl_xor_sync(0xFFFFFFFFu, wc, 1);
      we |= __shfl_xor_sync(0xFFFFFFFFu, we, 2);
      wc |= __shfl_xor_sync(0xFFFFFFFFu, wc, 2);
      const int64_t word = (tile << 3) + (lane >> 2);
      if ((lane & 3) == 0 && word < n_words) {
        flags[word] = we;
        flags[n_words + word] = wc;
      }
    }
  }
  if (err_first != nullptr && bad_min != INT64_MAX)
    atomicMin(reinterpret_cast<unsigned long long*>(err_first), (unsigned long long)bad_min);
}

// Scalar path (misaligned inputs): one query per thread, flags via ballot.
template <int KIND>
__global__ void __launch_bounds__(256) predict_scalar_kernel(
    const void* __restrict__ table, int64_t n_sig, const uint32_t* __restrict__ sig,
    const uint32_t* __restrict__ x, int64_t n_q, double* __restrict__ out,
    uint32_t* __restrict__ flags, int64_t* __restrict__ err_first) {
  constexpr int P = Planes<KIND>::P;
  const int64_t n_words = (n_q + 31) >> 5;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n_q; base += stride) {
    const int64_t q = base + threadIdx.x;
    bool e = false, c = false, bad = false;
    if (q < n_q) {
      uint32_t xs[P];
#pragma unroll
      for (int p = 0; p < P; ++p) xs[p] = x[p * n_q + q];
      out[q] = eval_query<KIND>(table, n_sig, sig[q], xs, e, c, bad);
      if (bad && err_first != nullptr)
        atomicMin(reinterpret_cast<unsigned long long*>(err_first), (unsigned long long)q);
    }
    const uint32_t be = __ballot_sync(0xFFFFFFFFu, e), bc = __ballot_sync(0xFFFFFFFFu, c);
    if (flags != nullptr && (threadIdx.x & 31) == 0 && q < n_q) {
      flags[q >> 5] = be;
      flags[n_words + (q >> 5)] = bc;
    }
  }
}

template <int KIND>
cudaError_t launch_predict_kind(const void* table, int64_t n_sig, const uint32_t* sig,
                                const uint32_t* x, int64_t n_q, double* out, uint32_t* flags,
                                int64_t* err_first, cudaStream_t stream, int n_sm) {
  if (n_q == 0) return cudaSuccess;
  const bool aligned = ((uintptr_t)sig % 32 == 0) && ((uintptr_t)x % 32 == 0) &&
                       ((uintptr_t)out % 32 == 0) && ((uintptr_t)table % 32 == 0) &&
                       (Planes<KIND>::P == 1 || n_q % 8 == 0);
  int per_sm = 0;
  if (aligned) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, predict_vec_kernel<KIND>, 256, 0);
    const int64_t tiles = (n_q + 255) / 256;
    int64_t blocks = (int64_t)n_sm * (per_sm > 0 ? per_sm : 4);
    const int64_t need = (tiles + 7) / 8;
    if (blocks > need) blocks = need;
    predict_vec_kernel<KIND><<<(unsigned)blocks, 256, 0, stream>>>(table, n_sig, sig, x, n_q,
                                                                    out, flags, err_first);
  } else {
    int64_t blocks = (n_q + 255) / 256;
    if (blocks > (int64_t)n_sm * 16) blocks = (int64_t)n_sm * 16;
    predict_scalar_kernel<KIND><<<(unsigned)blocks, 256, 0, stream>>>(table, n_sig, sig, x, n_q,
                                                                       out, flags, err_first);
  }
  return cudaGetLastError();
}

cudaError_t launch_predict(int kind, const void* table, int64_t n_sig, const uint32_t* sig,
                           const uint32_t* x, int64_t n_q, double* out, uint32_t* flags,
                           int64_t* err_first, cudaStream_t stream, int n_sm) {
  if (kind == DOOLY_KIND_AFFINE)
    return launch_predict_kind<DOOLY_KIND_AFFINE>(table, n_sig, sig, x, n_q, out, flags,
                                                  err_first, stream, n_sm);
  return launch_predict_kind<DOOLY_KIND_ATTN>(table, n_sig, sig, x, n_q, out, flags, err_first,
                                              stream, n_sm);
}

}  // namespace dooly
