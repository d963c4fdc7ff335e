// K3 — batched latency prediction (replaces predict).
//
// HBM-bound gather/evaluate/stream kernel.  Per query the algorithmic traffic
// is sig (4 B) + features (4 B per u32 plane) + latency out (8 B) + 2 flag bits;
// the regressor table row (32 B affine / 128 B attention) is an L2-resident
// gather.  Layout choices for B200:
//   * each lane owns 4 consecutive queries -> 16-B vector loads of sig and of
//     every feature plane, 2x16-B stores of the latencies (fully coalesced);
//   * UNROLL tiles per warp iteration so every lane has 2*(1+planes) 16-B
//     streaming loads in flight before its first dependent gather;
//   * flag bits are assembled with warp shuffles (no atomics, no byte stores):
//     lanes 8w..8w+7 own bit-word w of each 128-query tile;
//   * grid = resident CTAs x 148 SMs, grid-stride over 128-query tiles.
#include "common.cuh"

namespace dooly {

template <int KIND>
struct PredictIO {
  static constexpr int PLANES = KIND == DOOLY_KIND_ATTN ? 3 : 1;
};

template <int KIND>
__device__ __forceinline__ double predict_one(const void* table, int64_t n_sig, uint32_t s,
                                              const uint32_t* xs, bool& extrap, bool& clamped,
                                              bool& bad) {
  clamped = false;
  extrap = false;
  if (s >= (uint64_t)n_sig) {
    bad = true;
    return nan64();
  }
  if constexpr (KIND == DOOLY_KIND_AFFINE) {
    AffineRow r = load_affine(static_cast<const dooly_affine_row*>(table), s);
    if (!affine_valid(r)) {
      bad = true;
      return nan64();
    }
    extrap = xs[0] < r.lo || xs[0] > r.hi;
    return clamp_floor(eval_affine(r, xs[0]), clamped);
  } else {
    AttnRow r = load_attn(static_cast<const dooly_attn_row*>(table), s);
    if (!attn_valid(r)) {
      bad = true;
      return nan64();
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) extrap |= xs[k] < r.lo[k] || xs[k] > r.hi[k];
    return clamp_floor(eval_attn(r, xs[0], xs[1], xs[2]), clamped);
  }
}

// Vector path: n_q tiles of 128 queries, all pointers 16-B aligned.
template <int KIND, int UNROLL>
__global__ void __launch_bounds__(256) predict_vec_kernel(
    const void* __restrict__ table, int64_t n_sig, const uint32_t* __restrict__ sig,
    const uint32_t* __restrict__ x, int64_t n_q, double* __restrict__ out,
    uint32_t* __restrict__ flags, int64_t* __restrict__ err_first) {
  constexpr int P = PredictIO<KIND>::PLANES;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n_tiles = (n_q + 127) >> 7;
  const int64_t n_words = (n_q + 31) >> 5;
  int64_t bad_min = INT64_MAX;

  for (int64_t t0 = warp * UNROLL; t0 < n_tiles; t0 += n_warps * UNROLL) {
    uint4 sv[UNROLL];
    uint4 xv[UNROLL][P];
    // issue every streaming load of the UNROLL tiles first
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int64_t q = ((t0 + u) << 7) + lane * 4;
      if (q + 3 < n_q) {
        sv[u] = ld_stream_u4(sig + q);
#pragma unroll
        for (int p = 0; p < P; ++p) xv[u][p] = ld_stream_u4(x + p * n_q + q);
      } else {
        uint32_t s4[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
        uint32_t x4[P][4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const bool in = q + j < n_q;
#pragma unroll
          for (int p = 0; p < P; ++p) x4[p][j] = in ? x[p * n_q + q + j] : 0u;
          if (in) s4[j] = sig[q + j];
        }
        sv[u] = make_uint4(s4[0], s4[1], s4[2], s4[3]);
#pragma unroll
        for (int p = 0; p < P; ++p) xv[u][p] = make_uint4(x4[p][0], x4[p][1], x4[p][2], x4[p][3]);
      }
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int64_t tile = t0 + u;
      if (tile >= n_tiles) break;
      const int64_t q = (tile << 7) + lane * 4;
      const uint32_t s4[4] = {sv[u].x, sv[u].y, sv[u].z, sv[u].w};
      uint32_t xq[4][P];
#pragma unroll
      for (int p = 0; p < P; ++p) {
        xq[0][p] = xv[u][p].x;
        xq[1][p] = xv[u][p].y;
        xq[2][p] = xv[u][p].z;
        xq[3][p] = xv[u][p].w;
      }
      double r[4];
      uint32_t ebits = 0, cbits = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        bool e, c, bad = false;
        if (q + j < n_q) {
          r[j] = predict_one<KIND>(table, n_sig, s4[j], xq[j], e, c, bad);
          ebits |= (uint32_t)e << j;
          cbits |= (uint32_t)c << j;
          if (bad && q + j < bad_min) bad_min = q + j;
        } else {
          r[j] = 0.0;
        }
      }
      if (q + 3 < n_q) {
        st_stream_f64x2(out + q, r[0], r[1]);
        st_stream_f64x2(out + q + 2, r[2], r[3]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (q + j < n_q) out[q + j] = r[j];
      }
      if (flags != nullptr) {
        const int sh = 4 * (lane & 7);
        uint32_t we = ebits << sh, wc = cbits << sh;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
          we |= __shfl_xor_sync(0xFFFFFFFFu, we, o);
          wc |= __shfl_xor_sync(0xFFFFFFFFu, wc, o);
        }
        const int64_t word = (tile << 2) + (lane >> 3);
        if ((lane & 7) == 0 && word < n_words) {
          flags[word] = we;
          flags[n_words + word] = wc;
        }
      }
    }
  }
  if (err_first != nullptr && bad_min != INT64_MAX)
    atomicMin(reinterpret_cast<unsigned long long*>(err_first), (unsigned long long)bad_min);
}

// Scalar path (unaligned pointers): one query per thread, flags via ballot.
template <int KIND>
__global__ void __launch_bounds__(256) predict_scalar_kernel(
    const void* __restrict__ table, int64_t n_sig, const uint32_t* __restrict__ sig,
    const uint32_t* __restrict__ x, int64_t n_q, double* __restrict__ out,
    uint32_t* __restrict__ flags, int64_t* __restrict__ err_first) {
  constexpr int P = PredictIO<KIND>::PLANES;
  const int64_t n_words = (n_q + 31) >> 5;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n_q; base += stride) {
    const int64_t q = base + threadIdx.x;
    bool e = false, c = false, bad = false;
    if (q < n_q) {
      uint32_t xs[P];
#pragma unroll
      for (int p = 0; p < P; ++p) xs[p] = x[p * n_q + q];
      out[q] = predict_one<KIND>(table, n_sig, sig[q], xs, e, c, bad);
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
  constexpr int UNROLL = 2;
  const bool aligned = ((uintptr_t)sig % 16 == 0) && ((uintptr_t)x % 16 == 0) &&
                       ((uintptr_t)out % 16 == 0) &&
                       (PredictIO<KIND>::PLANES == 1 || n_q % 4 == 0);
  int per_sm = 0;
  if (aligned) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, predict_vec_kernel<KIND, UNROLL>,
                                                  256, 0);
    const int64_t tiles = (n_q + 127) / 128;
    int64_t blocks = (int64_t)n_sm * (per_sm > 0 ? per_sm : 4);
    const int64_t need = (tiles + 8 * UNROLL - 1) / (8 * UNROLL);
    if (blocks > need) blocks = need;
    predict_vec_kernel<KIND, UNROLL><<<(unsigned)blocks, 256, 0, stream>>>(
        table, n_sig, sig, x, n_q, out, flags, err_first);
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
