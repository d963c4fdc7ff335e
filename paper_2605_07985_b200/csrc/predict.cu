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
#include <cstdlib>
#include <cstring>

#include <cuda.h>

#include "common.cuh"

namespace dooly {

template <int KIND>
struct Planes {
  static constexpr int P = KIND == DOOLY_KIND_AFFINE ? 1 : 3;
};

static_assert(sizeof(dooly_attn_row96) == 96, "packed attention row must be 3 sectors");
static_assert(sizeof(dooly_attn_pack_header) == 96, "pack header must be one row");

// Box field layout of a packed attention table, read from its header once per
// thread (uniform across the grid; ok == false makes every query unknown).
struct PackInfo {
  uint64_t m0, m1, m2;
  uint32_t s1, s2;
  bool ok;
};

__device__ __forceinline__ PackInfo read_pack_header(const void* table, int64_t n_sig) {
  PackInfo pk{};
  const dooly_attn_pack_header* h = static_cast<const dooly_attn_pack_header*>(table);
  const uint32_t magic = __ldg(&h->magic), ok = __ldg(&h->ok);
  const uint32_t w0 = __ldg(&h->width[0]), w1 = __ldg(&h->width[1]), w2 = __ldg(&h->width[2]);
  pk.ok = magic == DOOLY_PACK_MAGIC && ok == 1u && __ldg(&h->n_sig) == n_sig &&
          w0 >= 1 && w1 >= 1 && w2 >= 1 && w0 + w1 + w2 <= 64;
  pk.m0 = (1ull << (w0 & 63)) - 1;
  pk.m1 = (1ull << (w1 & 63)) - 1;
  pk.m2 = (1ull << (w2 & 63)) - 1;
  pk.s1 = w0 & 63;
  pk.s2 = (w0 + w1) & 63;
  return pk;
}

// inv_scale of a packed row, recomputed exactly as oracle/sim.py inv_scale:
// RN(1 / hi) (correctly-rounded reciprocal == IEEE 1.0 / hi) or 1 when hi == 0.
__device__ __forceinline__ double inv_of(uint32_t hi) {
  return hi != 0u ? __drcp_rn((double)hi) : 1.0;
}

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

struct Row96 {  // folded serving row (include/dooly_b200.h dooly_attn_row96)
  double w[12];
  uint32_t lo[3], hi[3];
};

__device__ __forceinline__ void unpack_box(uint64_t lb, uint64_t hb, const PackInfo& pk,
                                           uint32_t* lo, uint32_t* hi) {
  lo[0] = (uint32_t)(lb & pk.m0);
  lo[1] = (uint32_t)((lb >> pk.s1) & pk.m1);
  lo[2] = (uint32_t)((lb >> pk.s2) & pk.m2);
  hi[0] = (uint32_t)(hb & pk.m0);
  hi[1] = (uint32_t)((hb >> pk.s1) & pk.m1);
  hi[2] = (uint32_t)((hb >> pk.s2) & pk.m2);
}

__device__ __forceinline__ Row96 gather_attn96(const dooly_attn_row96* t, uint32_t s,
                                               const PackInfo& pk) {
  const double* p = reinterpret_cast<const double*>(t + s);
  Row96 r;
  ld_row_256(p, r.w[0], r.w[1], r.w[2], r.w[3]);
  ld_row_256(p + 4, r.w[4], r.w[5], r.w[6], r.w[7]);
  ld_row_256(p + 8, r.w[8], r.w[9], r.w[10], r.w[11]);
  unpack_box((uint64_t)__double_as_longlong(r.w[4]), (uint64_t)__double_as_longlong(r.w[8]), pk,
             r.lo, r.hi);
  return r;
}

template <int KIND>
__device__ __forceinline__ double eval_query(const void* table, int64_t n_sig, uint32_t s,
                                             const uint32_t* xs, bool& extrap, bool& clamped,
                                             bool& bad, const PackInfo& pk) {
  extrap = clamped = false;
  if (s >= (uint64_t)n_sig) {
    bad = true;
    return nan64();
  }
  if constexpr (KIND == DOOLY_KIND_ATTN_PACKED) {
    const Row96 r = gather_attn96(static_cast<const dooly_attn_row96*>(table) + 1, s, pk);
    if (!(r.lo[0] <= r.hi[0])) {
      bad = true;
      return nan64();
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) extrap |= xs[k] < r.lo[k] || xs[k] > r.hi[k];
    return clamp_floor(eval_row96(r.w, xs[0], xs[1], xs[2]), clamped);
  } else if constexpr (KIND == DOOLY_KIND_AFFINE) {
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
  PackInfo pk{};
  if constexpr (KIND == DOOLY_KIND_ATTN_PACKED) {
    pk = read_pack_header(table, n_sig);
    if (!pk.ok) n_sig = 0;
  }
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
        r[j] = eval_query<KIND>(table, n_sig, sv.v[j], xs, e, c, bad, pk);
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

// Cooperative packed-attention path (DOOLY_KIND_ATTN_PACKED; opt-in, see
// predict_attn_mode).
//
// The row gather is L1TEX-wavefront-bound: a warp-wide LDG.256 costs one
// wavefront per distinct 128-B line, so one lane fetching its own 96-B row
// with three LDG.256 costs ~3 wavefronts per query (predict_vec_kernel).
// Here THREE lanes share a row: lane k of a group loads sector k, so one
// LDG.256 covers the whole rows of 10 queries (1.5 lines each on average).
// The serving row groups its folded coefficients by feature (common.cuh
// fold_row96), so lane k evaluates the partial sum s_k from its own sector
// and its own two feature planes (loaded in lane-rotated plane order: no
// selects), lane 2 adds the two partials it receives by shuffle, clamps and
// stores.  The box check is split the same way: lane 1 holds lo_bits and
// tests x < lo, lane 2 holds hi_bits and tests x > hi (one ballot combines
// them; one shuffle brings lo_0 for the fitted-row test).  Tiles are 160
// queries: 10 groups x 16 consecutive queries; lanes 30 and 31 idle.
constexpr int kCoopGroups = 10;
constexpr int kCoopPerGroup = 16;
constexpr int kCoopTile = kCoopGroups * kCoopPerGroup;  // 160 queries = 5 flag words

template <int MINB, int B>
__global__ void __launch_bounds__(256, MINB) predict_attn_coop_kernel(
    const void* __restrict__ table, int64_t n_sig, const uint32_t* __restrict__ sig,
    const uint32_t* __restrict__ x, int64_t n_q, double* __restrict__ out,
    uint32_t* __restrict__ flags, int64_t* __restrict__ err_first) {
  PackInfo pk = read_pack_header(table, n_sig);
  if (!pk.ok) n_sig = 0;
  const int lane = threadIdx.x & 31;
  const int g = lane / 3, k = lane - 3 * g;
  const bool act = g < kCoopGroups;
  const bool k0 = k == 0, k1 = k == 1, k2 = k == 2;
  const int kn = k2 ? 0 : k + 1, kt = k0 ? 2 : k - 1;  // planes of x_{k+1}, x_{k+2}
  // this lane's box fields (own / next / third feature) and the x < lo vs
  // x > hi orientation (lane 1 compares complements: x < lo <=> ~x > ~lo)
  auto shf = [&](int i) { return i == 0 ? 0u : i == 1 ? pk.s1 : pk.s2; };
  auto msk = [&](int i) { return i == 0 ? pk.m0 : i == 1 ? pk.m1 : pk.m2; };
  const uint32_t sh_o = shf(k), sh_n = shf(kn), sh_t = shf(kt);
  const uint64_t m_o = msk(k), m_n = msk(kn), m_t = msk(kt);
  const uint32_t flip = k1 ? 0xFFFFFFFFu : 0u;
  const double* rows =
      reinterpret_cast<const double*>(static_cast<const dooly_attn_row96*>(table) + 1) + 4 * k;
  const uint32_t* xo = x + (int64_t)k * n_q;
  const uint32_t* xn = x + (int64_t)kn * n_q;
  const uint32_t* xt = x + (int64_t)kt * n_q;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n_tiles = (n_q + kCoopTile - 1) / kCoopTile;
  const int64_t n_words = (n_q + 31) >> 5;
  const uint32_t nsig32 = n_sig > 0xFFFFFFFFll ? 0xFFFFFFFFu : (uint32_t)n_sig;
  const uint32_t all_u32 = n_sig > 0xFFFFFFFFll ? 1u : 0u;
  int64_t bad_min = INT64_MAX;

  for (int64_t tile = warp; tile < n_tiles; tile += n_warps) {
    const int64_t qg = tile * kCoopTile + g * kCoopPerGroup;
    uint32_t ebits = 0, cbits = 0;
#pragma unroll
    for (int h = 0; h < kCoopPerGroup / 8; ++h) {
      const int64_t qh = qg + 8 * h;
      const bool live = act && qh < n_q;  // n_q % 8 == 0: a half is all in or all out
      // branch-free: dead halves re-read query 0 and unknown signatures read
      // the header row; both are masked by `valid` (no divergence, so the
      // shuffles below need no reconvergence)
      const int64_t qs = live ? qh : 0;
      const U8 sv = ld_stream_256(sig + qs);
      const U8 vo = ld_stream_256(xo + qs);
      const U8 vn = ld_stream_256(xn + qs);
      const U8 vt = ld_stream_256(xt + qs);
      double res[8];
      uint32_t badbits = 0;
#pragma unroll
      for (int j0 = 0; j0 < 8; j0 += B) {
        double a[B][4];
#pragma unroll
        for (int j = 0; j < B; ++j) {
          const uint32_t sj = sv.v[j0 + j];
          // unknown rows read the header row (index -1), masked by `valid`
          const int64_t rj = ((sj < nsig32) | all_u32) ? (int64_t)sj : -1;
          ld_row_256(rows + 12 * rj, a[j][0], a[j][1], a[j][2], a[j][3]);
        }
#pragma unroll
        for (int j = 0; j < B; ++j) {
          const int q = j0 + j;
          const double part = sector_sum(k0 ? a[j][0] : 0.0, a[j][1], a[j][2], a[j][3],
                                         (double)vo.v[q], (double)vn.v[q]);
          const double s0 = __shfl_up_sync(0xFFFFFFFFu, part, 2);
          const double s1 = __shfl_up_sync(0xFFFFFFFFu, part, 1);
          // box: lanes 1 / 2 test their bound on all three features
          const uint64_t wb = (uint64_t)__double_as_longlong(a[j][0]);
          const uint32_t f0 = (uint32_t)(wb & pk.m0);
          // (bitwise, not short-circuit: no branches around the shuffles)
          const uint32_t out_any =
              (uint32_t)((vo.v[q] ^ flip) > ((uint32_t)((wb >> sh_o) & m_o) ^ flip)) |
              (uint32_t)((vn.v[q] ^ flip) > ((uint32_t)((wb >> sh_n) & m_n) ^ flip)) |
              (uint32_t)((vt.v[q] ^ flip) > ((uint32_t)((wb >> sh_t) & m_t) ^ flip));
          const uint32_t below = __ballot_sync(0xFFFFFFFFu, out_any != 0u);
          const uint32_t lo0 = __shfl_up_sync(0xFFFFFFFFu, f0, 1);
          // lane 2 finishes (other lanes' results are unused)
          const uint32_t valid = (uint32_t)live & ((uint32_t)(sv.v[q] < nsig32) | all_u32) &
                                 (uint32_t)(lo0 <= f0);
          const double sum = add(add(s0, s1), part);
          const uint32_t cl = (uint32_t)(sum < DOOLY_CLAMP_FLOOR);
          const double p = cl ? DOOLY_CLAMP_FLOOR : sum;
          const uint32_t e = valid & (out_any | ((below >> (lane - 1)) & 1u));
          res[q] = valid ? p : nan64();
          ebits |= e << (8 * h + q);
          cbits |= (valid & cl) << (8 * h + q);
          badbits |= (valid ^ 1u) << q;
        }
      }
      if (k2 && live && badbits != 0u) bad_min = min(bad_min, qh + (__ffs(badbits) - 1));
      if (k2 && live) {
        st_stream_256(out + qh, res[0], res[1], res[2], res[3]);
        st_stream_256(out + qh + 4, res[4], res[5], res[6], res[7]);
      }
    }
    if (flags != nullptr) {
      // group g holds the 16 bits of its queries; word w = groups 2w, 2w+1
      const uint32_t pe = __shfl_down_sync(0xFFFFFFFFu, ebits, 3);
      const uint32_t pc = __shfl_down_sync(0xFFFFFFFFu, cbits, 3);
      const int64_t word = tile * (kCoopTile / 32) + (g >> 1);
      if (k2 && act && (g & 1) == 0 && word < n_words) {
        flags[word] = (ebits & 0xFFFFu) | (pe << 16);
        flags[n_words + word] = (cbits & 0xFFFFu) | (pc << 16);
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
  PackInfo pk{};
  if constexpr (KIND == DOOLY_KIND_ATTN_PACKED) {
    pk = read_pack_header(table, n_sig);
    if (!pk.ok) n_sig = 0;
  }
  const int64_t n_words = (n_q + 31) >> 5;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n_q; base += stride) {
    const int64_t q = base + threadIdx.x;
    bool e = false, c = false, bad = false;
    if (q < n_q) {
      uint32_t xs[P];
#pragma unroll
      for (int p = 0; p < P; ++p) xs[p] = x[p * n_q + q];
      out[q] = eval_query<KIND>(table, n_sig, sig[q], xs, e, c, bad, pk);
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

// ---- staged packed-attention path (DOOLY_KIND_ATTN_PACKED; opt-in, measured
// slower than the one-lane kernel — profiles/r2_predict.md session 2).
//
// ncu on the one-lane-per-row kernel: the busiest unit is the L1 -> L2 request
// interface (l1tex__m_l1tex2xbar_req_cycles_active ~87%), and a lane's
// LDG.256 of one row sector is one request, so a 96-B row costs 3 requests.
// Here the warp fills its rows COOPERATIVELY with cp.async (LDGSTS, L2 ->
// shared memory without a register round trip): lane l copies 16-B chunk
// (l mod 6) of row (l / 6) in one instruction, so the 6 chunks of a row are
// adjacent lanes of the same instruction and coalesce into the 1-2 requests
// of the lines the row touches (~1.5 per row instead of 3).  Then every lane
// evaluates its own queries from shared memory with the one-lane arithmetic
// (eval_row96), so nothing is split across lanes.  Rows sit at a 112-B
// stride (7 x 16 B): LDS.128 by 8 consecutive lanes hits 8 distinct bank
// quads.  Steps of kStQ = 64 queries per warp (2 per lane); sig is staged in
// shared memory for the fill's row lookups.
constexpr int kStQ = 32;                  // queries per warp step (one per lane)
constexpr int kStStride = 112;            // bytes per staged row
constexpr int kStWarps = 4;
constexpr int kStPer = kStQ * 6 / 32;     // 16-B chunks per lane per step (6)

__global__ void __launch_bounds__(kStWarps * 32, 5) predict_attn_staged_kernel(
    const void* __restrict__ table, int64_t n_sig, const uint32_t* __restrict__ sig,
    const uint32_t* __restrict__ x, int64_t n_q, double* __restrict__ out,
    uint32_t* __restrict__ flags, int64_t* __restrict__ err_first) {
  // two row buffers per warp: step k+1's fill is in flight while step k evaluates
  __shared__ __align__(16) unsigned char rows_s[kStWarps][2][kStQ * kStStride];
  __shared__ uint32_t sig_s[kStWarps][2][kStQ];
  PackInfo pk = read_pack_header(table, n_sig);
  if (!pk.ok) n_sig = 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned char* rows_g = static_cast<const unsigned char*>(table) + 96;
  // this lane's chunks: c = lane + 32 i -> row c / 6, byte offset 16 (c % 6)
  int ch_row[kStPer];
  uint32_t ch_off[kStPer], ch_dst[kStPer];
#pragma unroll
  for (int i = 0; i < kStPer; ++i) {
    const int c = lane + 32 * i;
    ch_row[i] = c / 6;
    ch_off[i] = 16u * (uint32_t)(c % 6);
    ch_dst[i] = (uint32_t)(ch_row[i] * kStStride) + ch_off[i];
  }
  const uint32_t rs_base0 = (uint32_t)__cvta_generic_to_shared(rows_s[wid][0]);
  const uint32_t rs_base1 = (uint32_t)__cvta_generic_to_shared(rows_s[wid][1]);
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n_steps = (n_q + kStQ - 1) / kStQ;
  const int64_t n_words = (n_q + 31) >> 5;
  int64_t bad_min = INT64_MAX;

  uint32_t sv_n = 0, xv_n[3] = {0u, 0u, 0u};
  // stage step `st` (buffer b): sig + features into registers / smem, issue the fill
  auto stage = [&](int64_t st, int b) {
    const int64_t q = st * kStQ + lane;
    const bool in = q < n_q;
    sv_n = in ? __ldg(sig + q) : 0xFFFFFFFFu;
#pragma unroll
    for (int p = 0; p < 3; ++p) xv_n[p] = in ? __ldg(x + p * n_q + q) : 0u;
    sig_s[wid][b][lane] = sv_n;
    __syncwarp();
    const uint32_t base = b ? rs_base1 : rs_base0;
#pragma unroll
    for (int i = 0; i < kStPer; ++i) {
      const uint32_t s = sig_s[wid][b][ch_row[i]];
      if (s < (uint64_t)n_sig) {
        const unsigned char* src = rows_g + (int64_t)s * 96 + ch_off[i];
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(base + ch_dst[i]),
                     "l"(src)
                     : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  int64_t st = warp;
  if (st < n_steps) stage(st, 0);
  for (int b = 0; st < n_steps; st += n_warps, b ^= 1) {
    const uint32_t sv = sv_n, x0 = xv_n[0], x1 = xv_n[1], x2 = xv_n[2];
    const bool more = st + n_warps < n_steps;
    if (more) {
      stage(st + n_warps, b ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncwarp();
    const int64_t q = st * kStQ + lane;
    const double2* rp = reinterpret_cast<const double2*>(rows_s[wid][b] + lane * kStStride);
    double w[12];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const double2 v = rp[k];
      w[2 * k] = v.x;
      w[2 * k + 1] = v.y;
    }
    uint32_t lo[3], hi[3];
    unpack_box((uint64_t)__double_as_longlong(w[4]), (uint64_t)__double_as_longlong(w[8]), pk, lo,
               hi);
    const bool live = q < n_q;
    const bool valid = live && sv < (uint64_t)n_sig && lo[0] <= hi[0];
    bool cl = false;
    const double p = clamp_floor(eval_row96(w, x0, x1, x2), cl);
    const bool e = valid && (x0 < lo[0] || x0 > hi[0] || x1 < lo[1] || x1 > hi[1] ||
                             x2 < lo[2] || x2 > hi[2]);
    if (live) out[q] = valid ? p : nan64();
    if (live && !valid && q < bad_min) bad_min = q;
    const uint32_t be = __ballot_sync(0xFFFFFFFFu, e), bc = __ballot_sync(0xFFFFFFFFu, valid && cl);
    if (flags != nullptr && lane == 0 && st < n_words) {
      flags[st] = be;
      flags[n_words + st] = bc;
    }
    __syncwarp();   // buffer b is refilled two steps later
  }
  if (err_first != nullptr && bad_min != INT64_MAX)
    atomicMin(reinterpret_cast<unsigned long long*>(err_first), (unsigned long long)bad_min);
}

// ---- paired packed-attention path (DOOLY_KIND_ATTN_PACKED).
//
// The one-lane kernel is bound by the L1 -> L2 request interface: each lane's
// LDG.256 of a row sector is its own request, 3.26 per query.  Here two
// lanes serve two queries j, j+1 with three loads, arranged so that two of
// them fetch ADJACENT sectors of one row in the same instruction (which
// coalesce into one request unless the pair straddles a line):
//     load 1: A <- row j sector 0,   B <- row j   sector 1
//     load 2: A <- row j sector 2,   B <- row j+1 sector 0
//     load 3: A <- row j+1 sector 1, B <- row j+1 sector 2
// (~2.25 requests per query).  Each lane forms the per-feature partial sums
// s_k (A.19) of the three sectors it holds, one shuffle exchange hands each
// finishing lane the s_1 it lacks (A finishes j, B finishes j+1), and the
// lane holding a query's lo_bits reports its x < lo test and lo_0 to the
// finishing lane.  Every instruction is uniform across the two roles.
// Pairs own 8 consecutive queries (sig / feature streams as LDG.256, results
// regrouped so each lane stores 4 consecutive latencies as one STG.256);
// tiles are 16 pairs x 8 = 128 queries per warp.
__device__ __forceinline__ double u2d(uint32_t v) { return (double)v; }

struct U4q {
  uint32_t v[4];
};
__device__ __forceinline__ U4q ld_stream_128(const uint32_t* p) {
  U4q r;
  asm("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
      : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3])
      : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream_128(double* p, double a, double b) {
  asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1,%2};" ::"l"(p),
               "d"(a), "d"(b)
               : "memory");
}

// QPP = queries per pair (8: 128-query tiles, LDG.256 streams; 4: 64-query
// tiles, LDG.128 streams, fewer live registers -> more resident warps)
#ifndef PAIR_STRIDE_D
#define PAIR_STRIDE_D 12  // doubles per packed row slot (experiment: 16 = 128-B slots)
#endif

// One 16 x QPP-query tile of the paired path (shared by the paired kernel and
// the pair warps of the hybrid kernel).
template <int QPP>
__device__ __forceinline__ void pair_tile(int64_t tile, const double* __restrict__ rows,
                                          int64_t n_sig, const PackInfo& pk,
                                          const uint32_t* __restrict__ sig,
                                          const uint32_t* __restrict__ x, int64_t n_q,
                                          double* __restrict__ out, uint32_t* __restrict__ flags,
                                          int64_t n_words, int64_t& bad_min, int lane) {
  constexpr int TQ = 16 * QPP;  // queries per warp tile
  const int pr = lane >> 1;
  const bool B = (lane & 1) != 0;
  const int64_t qp = tile * TQ + QPP * pr;
  const bool live = qp < n_q;  // n_q % 8 == 0: a pair's queries are all in or all out
  const int64_t qs = live ? qp : 0;
  uint32_t sv[QPP], x0[QPP], x1[QPP], x2[QPP];
  if constexpr (QPP == 8) {
    const U8 a = ld_stream_256(sig + qs), b = ld_stream_256(x + qs),
             c = ld_stream_256(x + n_q + qs), d = ld_stream_256(x + 2 * n_q + qs);
#pragma unroll
    for (int j = 0; j < 8; ++j) sv[j] = a.v[j], x0[j] = b.v[j], x1[j] = c.v[j], x2[j] = d.v[j];
  } else {
    const U4q a = ld_stream_128(sig + qs), b = ld_stream_128(x + qs),
              c = ld_stream_128(x + n_q + qs), d = ld_stream_128(x + 2 * n_q + qs);
#pragma unroll
    for (int j = 0; j < 4; ++j) sv[j] = a.v[j], x0[j] = b.v[j], x1[j] = c.v[j], x2[j] = d.v[j];
  }
  double res[QPP / 2];
  uint32_t ebits = 0, cbits = 0;
#pragma unroll
  for (int j = 0; j < QPP; j += 2) {
    const uint32_t sa = sv[j], sb = sv[j + 1];
    const double* ra = sa < (uint64_t)n_sig ? rows + PAIR_STRIDE_D * (int64_t)sa : rows - PAIR_STRIDE_D;
    const double* rb = sb < (uint64_t)n_sig ? rows + PAIR_STRIDE_D * (int64_t)sb : rows - PAIR_STRIDE_D;
    double w1[4], w2[4], w3[4];
    ld_row_256(B ? ra + 4 : ra, w1[0], w1[1], w1[2], w1[3]);
    ld_row_256(B ? rb : ra + 8, w2[0], w2[1], w2[2], w2[3]);
    ld_row_256(B ? rb + 8 : rb + 4, w3[0], w3[1], w3[2], w3[3]);
    const uint32_t a0 = x0[j], a1 = x1[j], a2 = x2[j];
    const uint32_t b0 = x0[j + 1], b1 = x1[j + 1], b2 = x2[j + 1];
    // slot 1: A (j, s0: x0, x1) | B (j, s1: x1, x2)
    // slot 2: A (j, s2: x2, x0) | B (j+1, s0: x0, x1)
    // slot 3: A (j+1, s1: x1, x2) | B (j+1, s2: x2, x0)
    const double u1 = u2d(B ? a1 : a0), v1 = u2d(B ? a2 : a1);
    const double u2 = u2d(B ? b0 : a2), v2 = u2d(B ? b1 : a0);
    const double u3 = u2d(B ? b2 : b1), v3 = u2d(B ? b0 : b2);
    const double S1 = sector_sum(B ? 0.0 : w1[0], w1[1], w1[2], w1[3], u1, v1);
    const double S2 = sector_sum(B ? w2[0] : 0.0, w2[1], w2[2], w2[3], u2, v2);
    const double S3 = sector_sum(0.0, w3[1], w3[2], w3[3], u3, v3);
    // A needs s1(j) = B's S1; B needs s1(j+1) = A's S3
    const double got = __shfl_xor_sync(0xFFFFFFFFu, B ? S1 : S3, 1);
    const double sum = B ? add(add(S2, got), S3) : add(add(S1, got), S2);
    // box: the finishing lane holds hi_bits (A: slot 2 = sector 2 of j; B:
    // slot 3 = sector 2 of j+1); the partner holds lo_bits (B: slot 1 =
    // sector 1 of j; A: slot 3 = sector 1 of j+1) and tests x < lo for it
    const uint64_t hib = (uint64_t)__double_as_longlong(B ? w3[0] : w2[0]);
    const uint64_t lob = (uint64_t)__double_as_longlong(B ? w1[0] : w3[0]);
    const uint32_t p0 = B ? a0 : b0, p1 = B ? a1 : b1, p2 = B ? a2 : b2;   // partner's query
    const uint32_t l0 = (uint32_t)(lob & pk.m0), l1 = (uint32_t)((lob >> pk.s1) & pk.m1),
                   l2 = (uint32_t)((lob >> pk.s2) & pk.m2);
    const bool below_p = (p0 < l0) | (p1 < l1) | (p2 < l2);
    const uint32_t lo0 = __shfl_xor_sync(0xFFFFFFFFu, l0, 1);
    const uint32_t bel = __ballot_sync(0xFFFFFFFFu, below_p);
    const bool below = (bel >> (lane ^ 1)) & 1u;
    const uint32_t h0 = (uint32_t)(hib & pk.m0), h1 = (uint32_t)((hib >> pk.s1) & pk.m1),
                   h2 = (uint32_t)((hib >> pk.s2) & pk.m2);
    const uint32_t m0 = B ? b0 : a0, m1 = B ? b1 : a1, m2 = B ? b2 : a2;  // my query
    const bool above = (m0 > h0) | (m1 > h1) | (m2 > h2);
    const uint32_t my_sig = B ? sb : sa;
    const bool valid = live && my_sig < (uint64_t)n_sig && lo0 <= h0;
    bool cl = false;
    const double pv = clamp_floor(sum, cl);
    const int jm = j + (B ? 1 : 0);                 // my query's index in the pair's QPP
    res[j >> 1] = valid ? pv : nan64();
    ebits |= (uint32_t)(valid && (below || above)) << jm;
    cbits |= (uint32_t)(valid && cl) << jm;
    if (live && !valid && qp + jm < bad_min) bad_min = qp + jm;
  }
  // regroup: A holds the even queries, B the odd ones -> A the first half, B the second
  if constexpr (QPP == 8) {
    const double g1 = __shfl_xor_sync(0xFFFFFFFFu, B ? res[0] : res[2], 1);  // A<-p1, B<-p4
    const double g2 = __shfl_xor_sync(0xFFFFFFFFu, B ? res[1] : res[3], 1);  // A<-p3, B<-p6
    if (live) {
      if (B)
        st_stream_256(out + qp + 4, g1, res[2], g2, res[3]);
      else
        st_stream_256(out + qp, res[0], g1, res[1], g2);
    }
  } else {
    const double g1 = __shfl_xor_sync(0xFFFFFFFFu, B ? res[0] : res[1], 1);  // A<-p1, B<-p2
    if (live) {
      if (B)
        st_stream_128(out + qp + 2, g1, res[1]);
      else
        st_stream_128(out + qp, res[0], g1);
    }
  }
  if (flags != nullptr) {
    // a pair's QPP bits; 32 / QPP pairs per flag word
    uint32_t e8 = ebits | __shfl_xor_sync(0xFFFFFFFFu, ebits, 1);
    uint32_t c8 = cbits | __shfl_xor_sync(0xFFFFFFFFu, cbits, 1);
    constexpr int PPW = 32 / QPP;                   // pairs per word
    const int sh = QPP * (pr % PPW);
    e8 <<= sh;
    c8 <<= sh;
#pragma unroll
    for (int o = 2; o < 2 * PPW; o <<= 1) {
      e8 |= __shfl_xor_sync(0xFFFFFFFFu, e8, o);
      c8 |= __shfl_xor_sync(0xFFFFFFFFu, c8, o);
    }
    const int64_t word = tile * (TQ / 32) + pr / PPW;
    if ((lane & (2 * PPW - 1)) == 0 && word < n_words) {
      flags[word] = e8;
      flags[n_words + word] = c8;
    }
  }
}

template <int QPP, int MINB>
__global__ void __launch_bounds__(256, MINB) predict_attn_pair_kernel(
    const void* __restrict__ table, int64_t n_sig, const uint32_t* __restrict__ sig,
    const uint32_t* __restrict__ x, int64_t n_q, double* __restrict__ out,
    uint32_t* __restrict__ flags, int64_t* __restrict__ err_first) {
  constexpr int TQ = 16 * QPP;  // queries per warp tile
  PackInfo pk = read_pack_header(table, n_sig);
  if (!pk.ok) n_sig = 0;
  const int lane = threadIdx.x & 31;
  const double* rows = reinterpret_cast<const double*>(table) + PAIR_STRIDE_D;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n_tiles = (n_q + TQ - 1) / TQ;
  const int64_t n_words = (n_q + 31) >> 5;
  int64_t bad_min = INT64_MAX;
  for (int64_t tile = warp; tile < n_tiles; tile += n_warps)
    pair_tile<QPP>(tile, rows, n_sig, pk, sig, x, n_q, out, flags, n_words, bad_min, lane);
  if (err_first != nullptr && bad_min != INT64_MAX)
    atomicMin(reinterpret_cast<unsigned long long*>(err_first), (unsigned long long)bad_min);
}

// ---- hybrid packed-attention path (DOOLY_PREDICT_ATTN=hybrid).
//
// profiles/r2_predict.md session 5: TMA tile::gather4 row fetches and LDG.256
// row gathers do not share one request interface completely — warps of both
// kinds side by side gather ~14% more random 96-B rows per second than either
// alone.  Here NPW warps per CTA run the paired path over the first part of the
// query range and NTW warps serve the rest in 32-query rounds: lane l's row
// arrives in shared memory by `cp.async.bulk.tensor.2d ... tile::gather4`
// (lanes 0-7 each fetch the rows of lanes 4i..4i+3; one mbarrier per stage
// counts the 3 KB), HY_D stages in flight per warp, sig/features loaded into
// registers one round before the gather is issued.  The lane then evaluates
// its own query with the one-lane arithmetic (eval_row96), so every query's
// value and flags are those of the other paths bit for bit.
constexpr int HY_D = 3;                   // gather stages per TMA warp
constexpr int HY_STAGE = 32 * 96;         // bytes per stage (32 rows)

__device__ __forceinline__ void hy_wait(uint32_t bar, uint32_t parity) {
  // bounded: a byte-count mismatch must fail loudly, not hang the GPU
  for (uint32_t spin = 0;; ++spin) {
    uint32_t done;
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    if (spin > (1u << 26)) __trap();
  }
}

template <int NPW, int NTW>
__global__ void __launch_bounds__(32 * (NPW + NTW), 2) predict_attn_hybrid_kernel(
    const __grid_constant__ CUtensorMap tmap, const void* __restrict__ table, int64_t n_sig,
    const uint32_t* __restrict__ sig, const uint32_t* __restrict__ x, int64_t n_q,
    double* __restrict__ out, uint32_t* __restrict__ flags, int64_t* __restrict__ err_first,
    int64_t pair_q0) {
  extern __shared__ __align__(128) unsigned char hy_smem[];
  PackInfo pk = read_pack_header(table, n_sig);
  if (!pk.ok) n_sig = 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t n_words = (n_q + 31) >> 5;
  int64_t bad_min = INT64_MAX;
  if (wid < NPW) {
    // paired path over tiles [pair_q0 / 128, n_tiles)
    const double* rows =
        reinterpret_cast<const double*>(static_cast<const dooly_attn_row96*>(table) + 1);
    const int64_t n_tiles = (n_q + 127) / 128;
    const int64_t nw = (int64_t)gridDim.x * NPW;
    for (int64_t tile = pair_q0 / 128 + blockIdx.x * (int64_t)NPW + wid; tile < n_tiles; tile += nw)
      pair_tile<8>(tile, rows, n_sig, pk, sig, x, n_q, out, flags, n_words, bad_min, lane);
  } else {
    const int tw = wid - NPW;
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(hy_smem) + 8u * HY_D * tw;
    const uint32_t slot0 = (uint32_t)__cvta_generic_to_shared(hy_smem) + 128u * ((8 * HY_D * NTW + 127) / 128) +
                           (uint32_t)(HY_STAGE * HY_D * tw);
    const unsigned char* slot_p = hy_smem + 128 * ((8 * HY_D * NTW + 127) / 128) + HY_STAGE * HY_D * tw;
    if (lane == 0)
      for (int b = 0; b < HY_D; ++b)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8u * b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const int64_t n_rounds = pair_q0 / 32;          // the TMA range: queries [0, pair_q0)
    const int64_t nw = (int64_t)gridDim.x * NTW;
    const int64_t r0 = blockIdx.x * (int64_t)NTW + tw;
    // Software pipeline per warp (rounds rd, rd + nw, ... of this warp): the
    // sig of a round is loaded 4 rounds before its gather is issued, its
    // features when the gather is issued, and it is evaluated 2 rounds later.
    struct Q {
      uint32_t s, a, b, c;
    };
    auto ld_sig = [&](int64_t rd) {
      return rd < n_rounds ? __ldg(sig + rd * 32 + lane) : 0xFFFFFFFFu;
    };
    auto ld_x = [&](int64_t rd, uint32_t sv) {
      Q v{sv, 0u, 0u, 0u};
      if (rd < n_rounds) {
        const int64_t q = rd * 32 + lane;
        v.a = __ldg(x + q);
        v.b = __ldg(x + n_q + q);
        v.c = __ldg(x + 2 * n_q + q);
      }
      return v;
    };
    auto issue = [&](int64_t rd, uint32_t s, int b) {
      if (rd >= n_rounds) return;
      const int32_t row = s < (uint64_t)n_sig ? (int32_t)s + 1 : 0;   // row 0: the header
      const int i0 = (lane & 7) * 4;
      const int32_t g0 = __shfl_sync(0xFFFFFFFFu, row, i0), g1 = __shfl_sync(0xFFFFFFFFu, row, i0 + 1),
                    g2 = __shfl_sync(0xFFFFFFFFu, row, i0 + 2), g3 = __shfl_sync(0xFFFFFFFFu, row, i0 + 3);
      const uint32_t bar = bar0 + 8u * b;
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(HY_STAGE)
                     : "memory");
      __syncwarp();
      if (lane < 8)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(slot0 + (uint32_t)(HY_STAGE * b + lane * 4 * 96)),
            "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(0), "r"(g0), "r"(g1), "r"(g2), "r"(g3),
            "r"(bar)
            : "memory");
    };
    // prologue: rounds r0, r0 + nw gathered; sigs of r0 + 2 nw .. r0 + 5 nw loaded
    Q qc = ld_x(r0, ld_sig(r0));
    issue(r0, qc.s, 0);
    Q q1 = ld_x(r0 + nw, ld_sig(r0 + nw));
    issue(r0 + nw, q1.s, 1);
    uint32_t s2 = ld_sig(r0 + 2 * nw), s3 = ld_sig(r0 + 3 * nw), s4 = ld_sig(r0 + 4 * nw),
             s5 = ld_sig(r0 + 5 * nw);
    uint32_t phase = 0;
    int b = 0;
    for (int64_t rd = r0; rd < n_rounds; rd += nw) {
      // gather round rd + 2 nw into the stage freed by round rd - nw
      const int b2 = b == 0 ? 2 : b - 1;
      issue(rd + 2 * nw, s2, b2);
      const Q q2 = ld_x(rd + 2 * nw, s2);
      s2 = s3;
      s3 = s4;
      s4 = s5;
      s5 = ld_sig(rd + 6 * nw);
      hy_wait(bar0 + 8u * b, (phase >> b) & 1u);
      phase ^= 1u << b;
      const double2* rp = reinterpret_cast<const double2*>(slot_p + HY_STAGE * b + lane * 96);
      double w[12];
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const double2 v = rp[k];
        w[2 * k] = v.x;
        w[2 * k + 1] = v.y;
      }
      uint32_t lo[3], hi[3];
      unpack_box((uint64_t)__double_as_longlong(w[4]), (uint64_t)__double_as_longlong(w[8]), pk, lo,
                 hi);
      const int64_t q = rd * 32 + lane;
      const bool valid = qc.s < (uint64_t)n_sig && lo[0] <= hi[0];
      bool cl = false;
      const double pv = clamp_floor(eval_row96(w, qc.a, qc.b, qc.c), cl);
      const bool e = valid && (qc.a < lo[0] || qc.a > hi[0] || qc.b < lo[1] || qc.b > hi[1] ||
                               qc.c < lo[2] || qc.c > hi[2]);
      out[q] = valid ? pv : nan64();
      if (!valid && q < bad_min) bad_min = q;
      const uint32_t be = __ballot_sync(0xFFFFFFFFu, e), bc = __ballot_sync(0xFFFFFFFFu, valid && cl);
      if (flags != nullptr && lane == 0) {
        flags[rd] = be;
        flags[n_words + rd] = bc;
      }
      __syncwarp();   // stage b is re-filled by the next iteration's issue
      qc = q1;
      q1 = q2;
      b = b == 2 ? 0 : b + 1;
    }
  }
  if (err_first != nullptr && bad_min != INT64_MAX)
    atomicMin(reinterpret_cast<unsigned long long*>(err_first), (unsigned long long)bad_min);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// 2-D tensor map over the packed table's rows (header = row 0): 24 u32 words x
// (n_sig + 1) rows, 96-B row stride, box = one row.
static bool row96_tensor_map(CUtensorMap* m, const void* table, int64_t n_sig) {
  static EncodeTiledFn encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess)
      fn = nullptr;
    return reinterpret_cast<EncodeTiledFn>(fn);
  }();
  if (encode == nullptr || n_sig + 1 > (int64_t)INT32_MAX) return false;
  const cuuint64_t dims[2] = {24, (cuuint64_t)(n_sig + 1)};
  const cuuint64_t strides[1] = {96};
  const cuuint32_t box[2] = {24, 1};
  const cuuint32_t estr[2] = {1, 1};
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(table), dims, strides, box,
                estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// DOOLY_PREDICT_ATTN selects the packed-attention kernel: default the paired
// kernel (two lanes, two queries, three loads of which two coalesce: 2.5 L2
// requests per query, 93 G q/s at C5); "vec" one lane per row (3.26 requests,
// 81 G q/s); "staged" the cp.async-filled shared-memory variant (73 G q/s);
// "coop" / "coop8" / "coop1" the 3-lanes-per-row kernel (59 G q/s).  The
// request counts and why the others lose: profiles/r2_predict.md.
static int predict_attn_mode() {
  const char* v = getenv("DOOLY_PREDICT_ATTN");
  return v == nullptr              ? 5
         : strcmp(v, "coop") == 0  ? 0
         : strcmp(v, "coop8") == 0 ? 2
         : strcmp(v, "coop1") == 0 ? 3
         : strcmp(v, "staged") == 0 ? 4
         : strcmp(v, "vec") == 0 ? 1
         : strcmp(v, "pair4") == 0 ? 6
         : strcmp(v, "pair4b") == 0 ? 7
         : strcmp(v, "pair3") == 0 ? 8
         : strcmp(v, "hybrid") == 0 ? 9
                                   : 5;
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
  const int mode = predict_attn_mode();
  if (KIND == DOOLY_KIND_ATTN_PACKED && mode == 4 && (uintptr_t)table % 16 == 0) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, predict_attn_staged_kernel,
                                                  kStWarps * 32, 0);
    const int64_t steps = (n_q + kStQ - 1) / kStQ;
    int64_t blocks = (int64_t)n_sm * (per_sm > 0 ? per_sm : 1);
    const int64_t need = (steps + kStWarps - 1) / kStWarps;
    if (blocks > need) blocks = need;
    predict_attn_staged_kernel<<<(unsigned)blocks, kStWarps * 32, 0, stream>>>(
        table, n_sig, sig, x, n_q, out, flags, err_first);
  } else if (KIND == DOOLY_KIND_ATTN_PACKED && aligned && mode == 9 && n_q >= 128) {
    // TMA share of the queries (DOOLY_PREDICT_TMA_FRAC, default 0.3), whole 128-query tiles
    const char* fv = getenv("DOOLY_PREDICT_TMA_FRAC");
    const double frac = fv ? atof(fv) : 0.3;
    const int64_t n_tiles = (n_q + 127) / 128;
    int64_t tma_tiles = (int64_t)(frac * (double)n_tiles);
    if (tma_tiles < 0) tma_tiles = 0;
    if (tma_tiles > n_tiles - 1) tma_tiles = n_tiles - 1;
    CUtensorMap tm;
    if (!row96_tensor_map(&tm, table, n_sig)) return cudaErrorInvalidValue;
    constexpr int NPW = 8, NTW = 4;
    const size_t smem = 128 * ((8 * HY_D * NTW + 127) / 128) + (size_t)HY_STAGE * HY_D * NTW;
    auto kern = predict_attn_hybrid_kernel<NPW, NTW>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * (NPW + NTW), smem);
    const int64_t blocks = (int64_t)n_sm * (per_sm > 0 ? per_sm : 1);
    kern<<<(unsigned)blocks, 32 * (NPW + NTW), smem, stream>>>(tm, table, n_sig, sig, x, n_q, out,
                                                               flags, err_first, tma_tiles * 128);
  } else if (KIND == DOOLY_KIND_ATTN_PACKED && aligned && (mode >= 5 && mode <= 9)) {
    // (mode 9 below 128 queries: the paired kernel alone)
    auto kern = mode == 6 ? predict_attn_pair_kernel<4, 3>
              : mode == 7 ? predict_attn_pair_kernel<4, 2>
              : mode == 8 ? predict_attn_pair_kernel<8, 3> : predict_attn_pair_kernel<8, 2>;
    const int tq = (mode == 6 || mode == 7) ? 64 : 128;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
    const int64_t tiles = (n_q + tq - 1) / tq;
    int64_t blocks = (int64_t)n_sm * (per_sm > 0 ? per_sm : 1);
    const int64_t need = (tiles + 7) / 8;
    if (blocks > need) blocks = need;
    kern<<<(unsigned)blocks, 256, 0, stream>>>(table, n_sig, sig, x, n_q, out, flags, err_first);
  } else if (KIND == DOOLY_KIND_ATTN_PACKED && aligned && mode != 1 && mode != 4) {
    auto kern = mode == 2 ? predict_attn_coop_kernel<2, 8>
              : mode == 3 ? predict_attn_coop_kernel<1, 8>
                          : predict_attn_coop_kernel<2, 4>;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
    const int64_t tiles = (n_q + kCoopTile - 1) / kCoopTile;
    int64_t blocks = (int64_t)n_sm * (per_sm > 0 ? per_sm : 1);
    const int64_t need = (tiles + 7) / 8;
    if (blocks > need) blocks = need;
    kern<<<(unsigned)blocks, 256, 0, stream>>>(table, n_sig, sig, x, n_q, out, flags, err_first);
  } else if (aligned) {
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
  if (kind == DOOLY_KIND_ATTN_PACKED)
    return launch_predict_kind<DOOLY_KIND_ATTN_PACKED>(table, n_sig, sig, x, n_q, out, flags,
                                                       err_first, stream, n_sm);
  return launch_predict_kind<DOOLY_KIND_ATTN>(table, n_sig, sig, x, n_q, out, flags, err_first,
                                              stream, n_sm);
}

// ---- attention table -> packed predict form ------------------------------
// Pass 1: per-feature max of hi over fitted rows and a count of rows the
// packed form cannot represent exactly (inv_scale != 1/hi, or lo > hi in a
// feature) — block-reduced, one atomic per CTA per field.
__global__ void __launch_bounds__(256) attn_pack_scan_kernel(const dooly_attn_row* __restrict__ t,
                                                             int64_t n_sig,
                                                             dooly_attn_pack_header* h) {
  uint32_t mx[3] = {0u, 0u, 0u}, bad = 0u;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n_sig;
       s += (int64_t)gridDim.x * blockDim.x) {
    const AttnRow r = load_attn(t, (uint32_t)s);
    if (!attn_valid(r)) continue;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      mx[k] = max(mx[k], r.hi[k]);
      bad += (r.lo[k] > r.hi[k]) ||
             (__double_as_longlong(r.inv[k]) != __double_as_longlong(inv_of(r.hi[k])));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int k = 0; k < 3; ++k) mx[k] = max(mx[k], __shfl_xor_sync(0xFFFFFFFFu, mx[k], o));
    bad += __shfl_xor_sync(0xFFFFFFFFu, bad, o);
  }
  __shared__ uint32_t sm[8][4];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sm[w][0] = mx[0];
    sm[w][1] = mx[1];
    sm[w][2] = mx[2];
    sm[w][3] = bad;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    uint32_t v = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i)
      v = threadIdx.x == 3 ? v + sm[i][3] : max(v, sm[i][threadIdx.x]);
    if (threadIdx.x == 3) {
      if (v) atomicAdd(&h->bad_inv, v);
    } else if (v) {
      atomicMax(&h->max_hi[threadIdx.x], v);
    }
  }
}

// Pass 2: widths from the maxima, rows re-encoded; CTA 0 publishes the header.
__global__ void __launch_bounds__(256) attn_pack_write_kernel(const dooly_attn_row* __restrict__ t,
                                                              int64_t n_sig,
                                                              dooly_attn_pack_header* h) {
  uint32_t w[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) w[k] = max(1, 32 - __clz((int)h->max_hi[k]));
  const uint32_t s1 = w[0], s2 = w[0] + w[1];
  const bool fits = w[0] + w[1] + w[2] <= 64;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    h->width[0] = w[0];
    h->width[1] = w[1];
    h->width[2] = w[2];
    h->n_sig = n_sig;
    h->ok = (fits && h->bad_inv == 0u) ? 1u : 0u;
    h->magic = DOOLY_PACK_MAGIC;
  }
  dooly_attn_row96* out = reinterpret_cast<dooly_attn_row96*>(h) + 1;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n_sig;
       s += (int64_t)gridDim.x * blockDim.x) {
    const AttnRow r = load_attn(t, (uint32_t)s);
    uint64_t lb = ~0ull, hb = 0ull;
    if (attn_valid(r) && fits) {
      lb = (uint64_t)r.lo[0] | ((uint64_t)r.lo[1] << s1) | ((uint64_t)r.lo[2] << s2);
      hb = (uint64_t)r.hi[0] | ((uint64_t)r.hi[1] << s1) | ((uint64_t)r.hi[2] << s2);
    }
    double w[12];
    fold_row96(r.c, r.inv, lb, hb, w);
    double2* o = reinterpret_cast<double2*>(out + s);
#pragma unroll
    for (int i = 0; i < 6; ++i) o[i] = make_double2(w[2 * i], w[2 * i + 1]);
  }
}

cudaError_t launch_attn_pack(const void* table, int64_t n_sig, void* packed, cudaStream_t stream,
                             int n_sm, int64_t* launches) {
  dooly_attn_pack_header* h = static_cast<dooly_attn_pack_header*>(packed);
  cudaError_t e = cudaMemsetAsync(h, 0, sizeof(dooly_attn_pack_header), stream);
  if (e != cudaSuccess) return e;
  int64_t blocks = (n_sig + 255) / 256;
  if (blocks > (int64_t)n_sm * 8) blocks = (int64_t)n_sm * 8;
  if (blocks < 1) blocks = 1;
  const dooly_attn_row* t = static_cast<const dooly_attn_row*>(table);
  attn_pack_scan_kernel<<<(unsigned)blocks, 256, 0, stream>>>(t, n_sig, h);
  attn_pack_write_kernel<<<(unsigned)blocks, 256, 0, stream>>>(t, n_sig, h);
  *launches += 2;
  return cudaGetLastError();
}

}  // namespace dooly
