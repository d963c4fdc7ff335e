// Owner-routed multi-GPU dedup (SURVEY §8(e) dedup row): the routing,
// bucketing and global-uid steps of paper_2605_07985_b200/dist.py
// dedup_routed as device kernels — no eager tensor ops on the data path.
//
//   plan   owner(d) = (last 8 digest bytes as int64 & INT64_MAX) mod world;
//          a STABLE counting sort of the local digests by owner (per-block
//          histograms, a per-owner scan over blocks, then a ballot-ranked
//          scatter that keeps each bucket in record order), emitting the
//          permutation, the per-owner counts and the routed digests plus
//          their global indices in bucket order — ready for the all-to-all;
//   reply  on the owner, after dedup_digests + dedup_firsts: each received
//          record's global first index, its global uid (= number of first
//          occurrences, over ALL owners, with a smaller global index: one
//          lower_bound per owner's sorted first list) and its flags;
//   finish back home, the replies scattered through the plan's permutation
//          into first / uid / is_new / in_db.
// Every rank therefore resolves ~n / world keys, and the result equals the
// single-rank dedup of the whole list bit for bit.
#include "common.cuh"

namespace dooly {

constexpr int kRouteThreads = 256;
constexpr int kRouteTile = 2048;  // records per block (8 rounds of 256)
constexpr int kRouteMaxWorld = DOOLY_MAX_PEERS + 1;

__device__ __forceinline__ int owner_of(const uint8_t* digest, int world) {
  const uint64_t tail = *reinterpret_cast<const uint64_t*>(digest + 24) & 0x7FFFFFFFFFFFFFFFull;
  return (int)(tail % (uint64_t)world);
}

__global__ void __launch_bounds__(kRouteThreads) route_hist_kernel(const uint8_t* __restrict__ dig,
                                                                   int64_t n, int world,
                                                                   int32_t* __restrict__ hist) {
  __shared__ int32_t h[kRouteMaxWorld];
  if (threadIdx.x < world) h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t b0 = (int64_t)blockIdx.x * kRouteTile;
  for (int k = threadIdx.x; k < kRouteTile; k += kRouteThreads) {
    const int64_t i = b0 + k;
    if (i < n) atomicAdd(&h[owner_of(dig + i * 32, world)], 1);
  }
  __syncthreads();
  if (threadIdx.x < world) hist[(int64_t)blockIdx.x * world + threadIdx.x] = h[threadIdx.x];
}

// One thread per owner: exclusive scan over the blocks, then owner offsets.
__global__ void route_scan_kernel(int32_t* hist, int64_t n_blocks, int world,
                                  int64_t* __restrict__ base, int64_t* __restrict__ counts) {
  __shared__ int64_t tot[kRouteMaxWorld];
  const int w = threadIdx.x;
  int64_t run = 0;
  if (w < world) {
    for (int64_t b = 0; b < n_blocks; ++b) {
      base[b * world + w] = run;
      run += hist[b * world + w];
    }
    tot[w] = run;
    counts[w] = run;
  }
  __syncthreads();
  if (w < world) {
    int64_t start = 0;
    for (int v = 0; v < w; ++v) start += tot[v];
    for (int64_t b = 0; b < n_blocks; ++b) base[b * world + w] += start;
  }
}

__global__ void __launch_bounds__(kRouteThreads) route_scatter_kernel(
    const uint8_t* __restrict__ dig, int64_t n, int world, int64_t gidx0,
    const int64_t* __restrict__ base, int64_t* __restrict__ perm, uint8_t* __restrict__ out_dig,
    int64_t* __restrict__ out_gidx) {
  __shared__ int64_t run[kRouteMaxWorld];
  __shared__ int32_t wcnt[kRouteThreads / 32][kRouteMaxWorld];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x < world) run[threadIdx.x] = base[(int64_t)blockIdx.x * world + threadIdx.x];
  __syncthreads();
  const int64_t b0 = (int64_t)blockIdx.x * kRouteTile;
  for (int r = 0; r < kRouteTile; r += kRouteThreads) {  // rounds in record order
    const int64_t i = b0 + r + threadIdx.x;
    const bool in = i < n;
    const int own = in ? owner_of(dig + i * 32, world) : -1;
    uint32_t mine = 0, below = 0;
    for (int w = 0; w < world; ++w) {
      const uint32_t m = __ballot_sync(0xFFFFFFFFu, own == w);
      if (lane == 0) wcnt[wid][w] = __popc(m);
      if (own == w) {
        mine = m;
        below = __popc(m & ((1u << lane) - 1u));
      }
    }
    (void)mine;
    __syncthreads();
    if (in) {
      int64_t dst = run[own] + below;
      for (int v = 0; v < wid; ++v) dst += wcnt[v][own];
      perm[dst] = i;
      const uint4* src = reinterpret_cast<const uint4*>(dig + i * 32);
      uint4* d = reinterpret_cast<uint4*>(out_dig + dst * 32);
      d[0] = src[0];
      d[1] = src[1];
      out_gidx[dst] = gidx0 + i;
    }
    __syncthreads();
    if (threadIdx.x < world) {
      int64_t add = 0;
      for (int v = 0; v < kRouteThreads / 32; ++v) add += wcnt[v][threadIdx.x];
      run[threadIdx.x] += add;
    }
    __syncthreads();
  }
}

size_t route_workspace_size(int64_t n, int world) {
  const int64_t nb = (n + kRouteTile - 1) / kRouteTile;
  return (size_t)(nb > 0 ? nb : 1) * world * (sizeof(int32_t) + sizeof(int64_t)) + 256;
}

cudaError_t launch_route_plan(const uint8_t* dig, int64_t n, int world, int64_t gidx0,
                              int64_t* perm, int64_t* counts, uint8_t* out_dig, int64_t* out_gidx,
                              void* ws, cudaStream_t stream, int64_t* launches) {
  const int64_t nb = (n + kRouteTile - 1) / kRouteTile;
  if (n == 0) return cudaMemsetAsync(counts, 0, sizeof(int64_t) * world, stream);
  int64_t* base = static_cast<int64_t*>(ws);
  int32_t* hist = reinterpret_cast<int32_t*>(base + nb * world);
  route_hist_kernel<<<(unsigned)nb, kRouteThreads, 0, stream>>>(dig, n, world, hist);
  route_scan_kernel<<<1, 32, 0, stream>>>(hist, nb, world, base, counts);
  route_scatter_kernel<<<(unsigned)nb, kRouteThreads, 0, stream>>>(dig, n, world, gidx0, base,
                                                                  perm, out_dig, out_gidx);
  *launches += 3;
  return cudaGetLastError();
}

// Replies of an owner: row i = (global first index, global uid, is_new | in_db << 1).
__global__ void __launch_bounds__(kRouteThreads) route_reply_kernel(
    const int64_t* __restrict__ gidx, const int64_t* __restrict__ first,
    const uint8_t* __restrict__ is_new, const uint8_t* __restrict__ in_db, int64_t m,
    const int64_t* __restrict__ all_firsts, int64_t per, int world, int64_t* __restrict__ rows) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const int64_t g = gidx[first[i]];
    int64_t uid = 0;
    for (int o = 0; o < world; ++o) {  // lower_bound in owner o's sorted first list
      const int64_t* l = all_firsts + (int64_t)o * per;
      int64_t lo = 0, hi = per;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (l[mid] < g) lo = mid + 1;
        else hi = mid;
      }
      uid += lo;
    }
    rows[3 * i] = g;
    rows[3 * i + 1] = uid;
    rows[3 * i + 2] = (int64_t)is_new[i] | ((int64_t)(in_db ? in_db[i] : 0) << 1);
  }
}

cudaError_t launch_route_reply(const int64_t* gidx, const int64_t* first, const uint8_t* is_new,
                               const uint8_t* in_db, int64_t m, const int64_t* all_firsts,
                               int64_t per, int world, int64_t* rows, cudaStream_t stream,
                               int n_sm, int64_t* launches) {
  if (m == 0) return cudaSuccess;
  int64_t b = (m + kRouteThreads - 1) / kRouteThreads;
  if (b > (int64_t)n_sm * 8) b = (int64_t)n_sm * 8;
  route_reply_kernel<<<(unsigned)b, kRouteThreads, 0, stream>>>(gidx, first, is_new, in_db, m,
                                                                all_firsts, per, world, rows);
  *launches += 1;
  return cudaGetLastError();
}

__global__ void __launch_bounds__(kRouteThreads) route_finish_kernel(
    const int64_t* __restrict__ rows, const int64_t* __restrict__ perm, int64_t n,
    int64_t* __restrict__ out_first, uint32_t* __restrict__ out_uid,
    uint8_t* __restrict__ out_is_new, uint8_t* __restrict__ out_in_db) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t j = perm[i];
    const int64_t f = rows[3 * i + 2];
    out_first[j] = rows[3 * i];
    out_uid[j] = (uint32_t)rows[3 * i + 1];
    out_is_new[j] = (uint8_t)(f & 1);
    if (out_in_db) out_in_db[j] = (uint8_t)((f >> 1) & 1);
  }
}

cudaError_t launch_route_finish(const int64_t* rows, const int64_t* perm, int64_t n,
                                int64_t* out_first, uint32_t* out_uid, uint8_t* out_is_new,
                                uint8_t* out_in_db, cudaStream_t stream, int n_sm,
                                int64_t* launches) {
  if (n == 0) return cudaSuccess;
  int64_t b = (n + kRouteThreads - 1) / kRouteThreads;
  if (b > (int64_t)n_sm * 8) b = (int64_t)n_sm * 8;
  route_finish_kernel<<<(unsigned)b, kRouteThreads, 0, stream>>>(rows, perm, n, out_first,
                                                                 out_uid, out_is_new, out_in_db);
  *launches += 1;
  return cudaGetLastError();
}

}  // namespace dooly
