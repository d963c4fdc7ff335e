// K1b — first-occurrence signature dedup against the DB key set
// (replaces dedup; key lookup semantics of PAPER.md:333).
//
// Open-addressing table of 2^k u32 slots (load <= 0.5) keyed by the 256-bit
// digest.  A slot stores a record index; it is claimed with atomicCAS and
// then only ever holds indices of ONE digest, whose minimum is kept with
// atomicMin — so "first occurrence" is exact and schedule-independent
// (SURVEY H4).  DB digests are inserted first with indices n + j and mark
// their slot; a batch record's atomicMin then wins the slot (i < n <= n + j)
// while the DB mark stays.  Full-digest equality is always checked against
// the immutable digest arrays, never against slot contents.
// uids (rank among first occurrences, in index order) come from one
// exclusive scan of the first-occurrence flags.
#include <cstdlib>
#include <cstring>

#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace dooly {

constexpr uint32_t kEmpty = 0xFFFFFFFFu;
constexpr int DEDUP_THREADS = 256;

struct DedupWs {
  uint32_t* slots;
  uint8_t* mark;
  uint32_t* slot_of;
  uint32_t* first_flag;
  uint32_t* rank;
  void* cub_tmp;
  size_t cub_bytes;
  uint64_t cap;
};

static uint64_t table_cap(int64_t n, int64_t n_db) {
  uint64_t need = 2 * (uint64_t)(n + n_db);
  uint64_t cap = 1024;
  while (cap < need) cap <<= 1;
  return cap;
}

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

static size_t cub_scan_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                (int64_t)(n > 0 ? n : 1));
  return bytes;
}

static DedupWs carve(void* base, int64_t n, int64_t n_db) {
  DedupWs w;
  w.cap = table_cap(n, n_db);
  char* p = static_cast<char*>(base);
  w.slots = reinterpret_cast<uint32_t*>(p);
  p += align256(w.cap * 4);
  w.mark = reinterpret_cast<uint8_t*>(p);
  p += align256(w.cap);
  w.slot_of = reinterpret_cast<uint32_t*>(p);
  p += align256((size_t)n * 4);
  w.first_flag = reinterpret_cast<uint32_t*>(p);
  p += align256((size_t)n * 4);
  w.rank = reinterpret_cast<uint32_t*>(p);
  p += align256((size_t)n * 4);
  w.cub_tmp = p;
  w.cub_bytes = cub_scan_bytes(n);
  return w;
}

size_t dedup_workspace_size(int64_t n, int64_t n_db) {
  const uint64_t cap = table_cap(n, n_db);
  return align256(cap * 4) + align256(cap) + 3 * align256((size_t)n * 4) +
         align256(cub_scan_bytes(n)) + 256;
}

__device__ __forceinline__ void load_digest(const uint8_t* p, uint32_t d[8]) {
  const uint4* q = reinterpret_cast<const uint4*>(p);
  uint4 a = __ldg(q), b = __ldg(q + 1);
  d[0] = a.x; d[1] = a.y; d[2] = a.z; d[3] = a.w;
  d[4] = b.x; d[5] = b.y; d[6] = b.z; d[7] = b.w;
}

__device__ __forceinline__ bool digest_eq(const uint8_t* p, const uint32_t d[8]) {
  uint32_t e[8];
  load_digest(p, e);
  bool eq = true;
#pragma unroll
  for (int k = 0; k < 8; ++k) eq &= e[k] == d[k];
  return eq;
}

// Insert keys [0, m) of `keys` with slot values base + i.
__global__ void __launch_bounds__(DEDUP_THREADS) dedup_insert_kernel(
    const uint8_t* __restrict__ keys, int64_t m, uint32_t base, const uint8_t* __restrict__ batch,
    int64_t n, const uint8_t* __restrict__ db, uint32_t* slots, uint8_t* mark,
    uint32_t* slot_of, uint64_t mask, const uint32_t* __restrict__ grp) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    // grouped records (grp = each record's group minimum): only the minima
    // insert; the others share their minimum's digest and slot
    if (grp != nullptr && __ldg(grp + i) != (uint32_t)i) continue;
    uint32_t d[8];
    load_digest(keys + i * 32, d);
    const uint32_t me = base + (uint32_t)i;
    uint64_t slot = d[0] & mask;
    while (true) {
      const uint32_t cur = atomicCAS(slots + slot, kEmpty, me);
      if (cur == kEmpty) break;
      const uint8_t* other = cur < (uint32_t)n ? batch + (int64_t)cur * 32
                                               : db + (int64_t)(cur - (uint32_t)n) * 32;
      if (digest_eq(other, d)) {
        if (me < cur) atomicMin(slots + slot, me);
        break;
      }
      slot = (slot + 1) & mask;
    }
    if (slot_of != nullptr) slot_of[i] = (uint32_t)slot;
    else mark[slot] = 1;  // DB pass
  }
}

// Warp-cooperative form (SURVEY §8 north_star): 8-lane groups, one 256-bit key
// per group, lane k holding word k.  The group's key load is one coalesced
// 32-B sector (4 keys per warp instruction); the group leader claims the slot
// with atomicCAS and broadcasts the occupant; on a collision every lane loads
// word k of the occupant's digest and the group compares all 256 bits with one
// __all_sync.  Same slot protocol as dedup_insert_kernel, so the resulting
// table (and every output) is identical.  Selected with DOOLY_DEDUP_INSERT=group.
__global__ void __launch_bounds__(DEDUP_THREADS) dedup_insert_group_kernel(
    const uint8_t* __restrict__ keys, int64_t m, uint32_t base, const uint8_t* __restrict__ batch,
    int64_t n, const uint8_t* __restrict__ db, uint32_t* slots, uint8_t* mark,
    uint32_t* slot_of, uint64_t mask, const uint32_t* __restrict__ grp) {
  const int lane = threadIdx.x & 31, k = lane & 7, g0 = lane & ~7;
  const unsigned gmask = 0xFFu << g0;
  const int64_t stride = ((int64_t)gridDim.x * blockDim.x) >> 3;
  const uint32_t* kw = reinterpret_cast<const uint32_t*>(keys);
  const uint32_t* bw = reinterpret_cast<const uint32_t*>(batch);
  const uint32_t* dw = reinterpret_cast<const uint32_t*>(db);
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3; i < m; i += stride) {
    if (grp != nullptr && __ldg(grp + i) != (uint32_t)i) continue;   // group-uniform
    const uint32_t w = __ldg(kw + i * 8 + k);
    const uint32_t me = base + (uint32_t)i;
    uint64_t slot = __shfl_sync(gmask, w, g0) & mask;
    while (true) {
      uint32_t cur = 0;
      if (k == 0) cur = atomicCAS(slots + slot, kEmpty, me);
      cur = __shfl_sync(gmask, cur, g0);
      if (cur == kEmpty) break;
      const uint32_t o = cur < (uint32_t)n ? __ldg(bw + (int64_t)cur * 8 + k)
                                           : __ldg(dw + (int64_t)(cur - (uint32_t)n) * 8 + k);
      if (__all_sync(gmask, o == w)) {
        if (k == 0 && me < cur) atomicMin(slots + slot, me);
        break;
      }
      slot = (slot + 1) & mask;
    }
    if (k == 0) {
      if (slot_of != nullptr) slot_of[i] = (uint32_t)slot;
      else mark[slot] = 1;  // DB pass
    }
  }
}

static bool dedup_group_insert() {
  const char* v = getenv("DOOLY_DEDUP_INSERT");
  return v != nullptr && strcmp(v, "group") == 0;
}

__global__ void __launch_bounds__(DEDUP_THREADS) dedup_resolve_kernel(
    int64_t n, const uint32_t* __restrict__ slots, const uint8_t* __restrict__ mark,
    const uint32_t* __restrict__ slot_of, int64_t* __restrict__ out_first,
    uint8_t* __restrict__ out_is_new, uint8_t* __restrict__ out_in_db, uint32_t* first_flag,
    const uint32_t* __restrict__ grp) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t s = slot_of[grp != nullptr ? __ldg(grp + i) : (uint32_t)i];
    const uint32_t f = slots[s];
    const uint8_t in_db = mark[s];
    const bool first = f == (uint32_t)i;
    out_first[i] = f;
    out_is_new[i] = (first && !in_db) ? 1 : 0;
    if (out_in_db) out_in_db[i] = in_db;
    first_flag[i] = first ? 1u : 0u;
  }
}

__global__ void __launch_bounds__(DEDUP_THREADS) dedup_uid_kernel(
    int64_t n, const int64_t* __restrict__ out_first, const uint32_t* __restrict__ rank,
    const uint32_t* __restrict__ first_flag, uint32_t* __restrict__ out_uid,
    int64_t* __restrict__ out_n_unique) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    out_uid[i] = rank[out_first[i]];
    if (i == n - 1) *out_n_unique = (int64_t)rank[i] + first_flag[i];
  }
}

static unsigned grid_for(int64_t m, int n_sm) {
  int64_t b = (m + DEDUP_THREADS - 1) / DEDUP_THREADS;
  const int64_t cap = (int64_t)n_sm * 8;
  if (b > cap) b = cap;
  return (unsigned)(b > 0 ? b : 1);
}

cudaError_t launch_dedup(const uint8_t* digests, int64_t n, const uint8_t* db, int64_t n_db,
                         int64_t* out_first, uint32_t* out_uid, uint8_t* out_is_new,
                         uint8_t* out_in_db, int64_t* out_n_unique, void* ws, size_t ws_bytes,
                         cudaStream_t stream, int n_sm, int64_t* launches,
                         const uint32_t* grp) {
  (void)ws_bytes;
  cudaError_t e;
  if (n == 0) return cudaMemsetAsync(out_n_unique, 0, sizeof(int64_t), stream);
  DedupWs w = carve(ws, n, n_db);
  if ((e = cudaMemsetAsync(w.slots, 0xFF, w.cap * 4, stream)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(w.mark, 0, w.cap, stream)) != cudaSuccess) return e;
  const uint64_t mask = w.cap - 1;
  const bool lanes8 = dedup_group_insert();
  auto insert = lanes8 ? dedup_insert_group_kernel : dedup_insert_kernel;
  auto grid = [&](int64_t m) { return grid_for(lanes8 ? 8 * m : m, n_sm); };
  if (n_db > 0) {
    insert<<<grid(n_db), DEDUP_THREADS, 0, stream>>>(db, n_db, (uint32_t)n, digests, n, db,
                                                     w.slots, w.mark, nullptr, mask, nullptr);
    *launches += 1;
  }
  insert<<<grid(n), DEDUP_THREADS, 0, stream>>>(digests, n, 0u, digests, n, db, w.slots, w.mark,
                                                w.slot_of, mask, grp);
  dedup_resolve_kernel<<<grid_for(n, n_sm), DEDUP_THREADS, 0, stream>>>(
      n, w.slots, w.mark, w.slot_of, out_first, out_is_new, out_in_db, w.first_flag, grp);
  size_t tmp = w.cub_bytes;
  if ((e = cub::DeviceScan::ExclusiveSum(w.cub_tmp, tmp, w.first_flag, w.rank, (int64_t)n,
                                         stream)) != cudaSuccess)
    return e;
  dedup_uid_kernel<<<grid_for(n, n_sm), DEDUP_THREADS, 0, stream>>>(
      n, out_first, w.rank, w.first_flag, out_uid, out_n_unique);
  *launches += 4;  // insert, resolve, cub scan, uid
  return cudaGetLastError();
}

// Owner-routed dedup (route.cu): after launch_dedup on an owner's received
// digests, the owner's first occurrences in order — out_firsts[rank[i]] =
// gidx[i] for every first occurrence i — read from the same workspace's
// first-occurrence flags and their exclusive scan.
__global__ void __launch_bounds__(DEDUP_THREADS) dedup_firsts_kernel(
    int64_t n, const uint32_t* __restrict__ first_flag, const uint32_t* __restrict__ rank,
    const int64_t* __restrict__ gidx, int64_t* __restrict__ out_firsts) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    if (first_flag[i]) out_firsts[rank[i]] = gidx[i];
}

// ---- record grouping ahead of SHA-256 (dooly_dedup): records whose packed
// content is identical apart from the repeat count (w3, not part of the
// canonical message, include/dooly_b200.h) have identical canonical bytes and
// therefore identical digests, so SHA-256 runs once per distinct content and
// the other records copy the representative's digest.  Exactness never rests
// on the 64-bit content hash: a slot stores a record index (claimed by CAS)
// and equality is decided by comparing the two records word by word.  Equal
// packed content is sufficient, not necessary, for equal digests; the digest
// dedup that follows still decides first occurrences over all records.
// The workspace is the digest dedup's own (slots, slot_of, rank, mark),
// consumed here before dooly_dedup_digests re-initialises it.
__device__ __forceinline__ uint64_t grp_mix(uint64_t h, uint32_t w) {
  return (h ^ w) * 0x100000001b3ull;
}
__device__ __forceinline__ uint64_t grp_fmix(uint64_t h) {
  h ^= h >> 33;
  h *= 0xff51afd7ed558ccdull;
  h ^= h >> 33;
  h *= 0xc4ceb9fe1a85ec53ull;
  return h ^ (h >> 33);
}

// Record length in words from its header: 4 + 3 n_dims + n_sym.
__device__ __forceinline__ uint32_t grp_len(const uint32_t* r) {
  const uint32_t w1 = __ldg(r + 1);
  return 4u + 3u * (w1 & 0xFFFFu) + (w1 >> 16);
}

// One thread per record.  Every load of a probe is independent of the
// others (no early exit inside the word loops), so a record costs a few
// memory round trips: its offset, its words, its slot, then either the CAS or
// the representative's offset and words.
__global__ void __launch_bounds__(DEDUP_THREADS) rec_group_kernel(
    const uint32_t* __restrict__ words, const int64_t* __restrict__ rec_off, int64_t n,
    uint32_t* slots, uint64_t mask, uint32_t* __restrict__ rep) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    {
      const uint32_t* r = words + rec_off[i];
      const uint32_t len = grp_len(r);
      uint64_t h = 0xcbf29ce484222325ull ^ len;
#pragma unroll 4
      for (uint32_t k = 0; k < len; ++k) {
        const uint32_t w = __ldg(r + k);
        h = k != 3 ? grp_mix(h, w) : h;
      }
      h = grp_fmix(h);
      uint64_t slot = h & mask;
      while (true) {
        uint32_t v = *reinterpret_cast<volatile uint32_t*>(slots + slot);
        if (v == kEmpty) {
          v = atomicCAS(slots + slot, kEmpty, (uint32_t)i);
          if (v == kEmpty) {
            rep[i] = (uint32_t)slot;   // the group's slot; rec_group_min_kernel resolves it
            break;
          }
        }
        // full comparison against the slot's representative v (repeat word excluded)
        const uint32_t* rv = words + rec_off[v];
        uint32_t diff = grp_len(rv) ^ len;
        if (diff == 0) {
#pragma unroll 4
          for (uint32_t k = 0; k < len; ++k)
            diff |= k != 3 ? (__ldg(rv + k) ^ __ldg(r + k)) : 0u;
        }
        if (diff == 0) {   // same content: the slot keeps the group's smallest index
          if ((uint32_t)i < v) atomicMin(slots + slot, (uint32_t)i);
          rep[i] = (uint32_t)slot;
          break;
        }
        slot = (slot + 1) & mask;
      }
    }
  }
}

// Each record's representative is its group's smallest index (the slot's
// final value); the representatives are listed for SHA-256.
__global__ void __launch_bounds__(DEDUP_THREADS) rec_group_min_kernel(
    const uint32_t* __restrict__ slots, int64_t n, uint32_t* __restrict__ rep,
    uint32_t* __restrict__ list, uint32_t* count) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // warp-uniform trip count (the list append is warp-aggregated)
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < n;
       base += stride) {
    const int64_t i = base + lane;
    bool is_rep = false;
    if (i < n) {
      const uint32_t m = slots[rep[i]];
      rep[i] = m;
      is_rep = m == (uint32_t)i;
    }
    const uint32_t b = __ballot_sync(0xFFFFFFFFu, is_rep);
    uint32_t at = 0;
    if (lane == 0 && b != 0u) at = atomicAdd(count, (uint32_t)__popc(b));
    at = __shfl_sync(0xFFFFFFFFu, at, 0);
    if (is_rep) list[at + __popc(b & ((1u << lane) - 1u))] = (uint32_t)i;
  }
}

__global__ void __launch_bounds__(DEDUP_THREADS) digest_copy_kernel(
    const uint32_t* __restrict__ rep, int64_t n, uint8_t* digests) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t r = rep[i];
    if (r != (uint32_t)i) {
      const uint4* src = reinterpret_cast<const uint4*>(digests + (int64_t)r * 32);
      uint4* dst = reinterpret_cast<uint4*>(digests + i * 32);
      dst[0] = src[0];
      dst[1] = src[1];
    }
  }
}

// rep lives in the scan's rank array (read by the digest copy and by the
// grouped insert / resolve, all before the scan), the list in slot_of (read by
// SHA-256 before the insert writes it), the count in the DB-mark bytes.
RecGroup rec_group_carve(void* ws, int64_t n, int64_t n_db) {
  DedupWs w = carve(ws, n, n_db);
  return RecGroup{w.rank, w.slot_of, reinterpret_cast<uint32_t*>(w.mark)};
}

cudaError_t launch_rec_group(const uint32_t* words, const int64_t* rec_off, int64_t n, void* ws,
                             int64_t n_db, cudaStream_t stream, int n_sm, int64_t* launches) {
  if (n == 0) return cudaSuccess;
  DedupWs w = carve(ws, n, n_db);
  const RecGroup g = rec_group_carve(ws, n, n_db);
  cudaError_t e;
  if ((e = cudaMemsetAsync(w.slots, 0xFF, w.cap * 4, stream)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(g.count, 0, sizeof(uint32_t), stream)) != cudaSuccess) return e;
  rec_group_kernel<<<grid_for(n, n_sm), DEDUP_THREADS, 0, stream>>>(words, rec_off, n, w.slots,
                                                                   w.cap - 1, g.rep);
  rec_group_min_kernel<<<grid_for(n, n_sm), DEDUP_THREADS, 0, stream>>>(w.slots, n, g.rep, g.list,
                                                                       g.count);
  *launches += 2;
  return cudaGetLastError();
}

cudaError_t launch_digest_copy(const uint32_t* rep, int64_t n, uint8_t* digests,
                               cudaStream_t stream, int n_sm, int64_t* launches) {
  if (n == 0) return cudaSuccess;
  digest_copy_kernel<<<grid_for(n, n_sm), DEDUP_THREADS, 0, stream>>>(rep, n, digests);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_dedup_firsts(int64_t n, int64_t n_db, const int64_t* gidx, int64_t* out_firsts,
                                void* ws, cudaStream_t stream, int n_sm, int64_t* launches) {
  if (n == 0) return cudaSuccess;
  DedupWs w = carve(ws, n, n_db);
  dedup_firsts_kernel<<<grid_for(n, n_sm), DEDUP_THREADS, 0, stream>>>(n, w.first_flag, w.rank,
                                                                       gidx, out_firsts);
  *launches += 1;
  return cudaGetLastError();
}

}  // namespace dooly
