// K1a — canonical serialisation + SHA-256 of packed operation records
// (replaces canonicalize, and signature_hash).
//
// One thread per record.  The canonical `sigfmt=1` message (layout pinned in
// SURVEY.md App. A.1 and restated in oracle/profiler.py) is rebuilt from the
// packed record + the op-name / kernel-symbol / attr-digest tables straight
// into a per-thread shared-memory block buffer as big-endian words (the
// message is never materialised in HBM).  Compression then runs block by
// block with all lanes of a warp in lock-step, so lanes whose messages have
// different lengths do not serialise each other mid-stream.  SHA-256 is pure
// 32-bit integer work (rotates, Ch/Maj via LOP3, adds): the kernel is bound by
// the integer pipes, not HBM.
#include "common.cuh"

namespace dooly {

__constant__ uint32_t kSha256K[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4,
    0xab1c5ed5, 0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe,
    0x9bdc06a7, 0xc19bf174, 0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f,
    0x4a7484aa, 0x5cb0a9dc, 0x76f988da, 0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7,
    0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967, 0x27b70a85, 0x2e1b2138, 0x4d2c6dfc,
    0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85, 0xa2bfe8a1, 0xa81a664b,
    0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070, 0x19a4c116,
    0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7,
    0xc67178f2};

__device__ __forceinline__ uint32_t rotr(uint32_t x, int n) { return __funnelshift_r(x, x, n); }
__device__ __forceinline__ uint32_t fadd(uint32_t a, uint32_t b, uint32_t one) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(one), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// One 64-byte block; w points at 16 big-endian words in shared memory.
// 16 rounds are unrolled (the a..h roles rotate back every 8 rounds) inside a
// 4-trip loop: ncu showed the fully unrolled 64-round body, inlined at two call
// sites, thrashing the instruction cache (`no_instruction` was the top stall).
#define SHA_S0(x) (rotr(x, 2) ^ rotr(x, 13) ^ rotr(x, 22))
#define SHA_S1(x) (rotr(x, 6) ^ rotr(x, 11) ^ rotr(x, 25))
#define SHA_s0(x) (rotr(x, 7) ^ rotr(x, 18) ^ ((x) >> 3))
#define SHA_s1(x) (rotr(x, 17) ^ rotr(x, 19) ^ ((x) >> 10))
// Pipe balance: the rotates (SHF) and Ch/Maj/xor (LOP3) can only run on the
// ALU pipe, which is what bounds SHA-256 (18 ALU instructions per round).  The
// 10 additions per round go to the FMA pipe instead, as IMAD a * one + b with
// `one` a kernel argument ptxas cannot fold back into IADD3.
#define SHA_ADD(x, y) fadd((x), (y), one)
#define SHA_RND(a, b, c, d, e, f, g, h, i)                                                   \
  {                                                                                          \
    const uint32_t t1 = SHA_ADD(SHA_ADD(SHA_ADD(h, SHA_S1(e)), (e & f) ^ (~e & g)),           \
                                SHA_ADD(kSha256K[r + i], w[i]));                             \
    const uint32_t t2 = SHA_ADD(SHA_S0(a), (a & b) ^ (a & c) ^ (b & c));                     \
    d = SHA_ADD(d, t1);                                                                      \
    h = SHA_ADD(t1, t2);                                                                     \
  }
#define SHA_SCHED(i)                                                                           \
  w[i] = SHA_ADD(SHA_ADD(SHA_ADD(w[i], SHA_s0(w[((i) + 1) & 15])), w[((i) + 9) & 15]),         \
                 SHA_s1(w[((i) + 14) & 15]))
#define SHA_16(sched)                                                              \
  sched(0); SHA_RND(a, b, c, d, e, f, g, k, 0);                                    \
  sched(1); SHA_RND(k, a, b, c, d, e, f, g, 1);                                    \
  sched(2); SHA_RND(g, k, a, b, c, d, e, f, 2);                                    \
  sched(3); SHA_RND(f, g, k, a, b, c, d, e, 3);                                    \
  sched(4); SHA_RND(e, f, g, k, a, b, c, d, 4);                                    \
  sched(5); SHA_RND(d, e, f, g, k, a, b, c, 5);                                    \
  sched(6); SHA_RND(c, d, e, f, g, k, a, b, 6);                                    \
  sched(7); SHA_RND(b, c, d, e, f, g, k, a, 7);                                    \
  sched(8); SHA_RND(a, b, c, d, e, f, g, k, 8);                                    \
  sched(9); SHA_RND(k, a, b, c, d, e, f, g, 9);                                    \
  sched(10); SHA_RND(g, k, a, b, c, d, e, f, 10);                                  \
  sched(11); SHA_RND(f, g, k, a, b, c, d, e, 11);                                  \
  sched(12); SHA_RND(e, f, g, k, a, b, c, d, 12);                                  \
  sched(13); SHA_RND(d, e, f, g, k, a, b, c, 13);                                  \
  sched(14); SHA_RND(c, d, e, f, g, k, a, b, 14);                                  \
  sched(15); SHA_RND(b, c, d, e, f, g, k, a, 15);
#define SHA_NOSCHED(i) (void)0

__device__ __forceinline__ void sha256_compress(uint32_t hs[8], const uint32_t* w_in,
                                                uint32_t one) {
  uint32_t w[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) w[i] = w_in[i];
  uint32_t a = hs[0], b = hs[1], c = hs[2], d = hs[3], e = hs[4], f = hs[5], g = hs[6],
           k = hs[7];
  int r = 0;
  SHA_16(SHA_NOSCHED)
#pragma unroll 1
  for (r = 16; r < 64; r += 16) {
    SHA_16(SHA_SCHED)
  }
  hs[0] += a;
  hs[1] += b;
  hs[2] += c;
  hs[3] += d;
  hs[4] += e;
  hs[5] += f;
  hs[6] += g;
  hs[7] += k;
}

// Out-of-line copy for the rare long-message drain inside the byte writer.
__device__ __noinline__ void sha256_compress_blocks(uint32_t hs[8], const uint32_t* w, int nb) {
  for (int b = 0; b < nb; ++b) sha256_compress(hs, w + 16 * b, 1u);
}

constexpr int SHA_THREADS = 128;
#ifndef SHA_MINB
#define SHA_MINB 4  // 4M C5 records: 0.831 ms at 4 CTAs/SM (88 registers), 0.833 at 5, 0.846 at 6, 0.854 at 7
#endif
constexpr int SHA_BUF_BLOCKS = 3;  // 192 B: C1-C5 canonical messages fit (longer ones drain)
constexpr int SHA_STRIDE = SHA_BUF_BLOCKS * 16 + 1;   // odd word stride: conflict-free reads

// Byte-stream writer into a per-thread shared-memory block buffer.
struct ShaStream {
  uint32_t* buf;
  uint32_t h[8];
  uint32_t pend;  // pending bytes, high-aligned
  int pn;         // pending byte count (0..3)
  int nw;         // complete words in buf
  uint64_t total; // message bytes

  __device__ void init(uint32_t* b) {
    buf = b;
    h[0] = 0x6a09e667;
    h[1] = 0xbb67ae85;
    h[2] = 0x3c6ef372;
    h[3] = 0xa54ff53a;
    h[4] = 0x510e527f;
    h[5] = 0x9b05688c;
    h[6] = 0x1f83d9ab;
    h[7] = 0x5be0cd19;
    pend = 0;
    pn = 0;
    nw = 0;
    total = 0;
  }
  __device__ __forceinline__ void emit(uint32_t w) {
    buf[nw++] = w;
    if (nw == SHA_BUF_BLOCKS * 16) {  // long message: drain (rare, divergent)
      // The out-of-line drain gets a COPY of the chaining state: passing h
      // itself would take its address and force the whole stream state into
      // local memory (an LDL/STL pair around every emitted byte and word).
      uint32_t t[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) t[k] = h[k];
      sha256_compress_blocks(t, buf, SHA_BUF_BLOCKS);
#pragma unroll
      for (int k = 0; k < 8; ++k) h[k] = t[k];
      nw = 0;
    }
  }
  __device__ __forceinline__ void put_be32(uint32_t c) {
    total += 4;
    if (pn == 0) {
      emit(c);
    } else {
      emit(pend | (c >> (8 * pn)));
      pend = c << (32 - 8 * pn);
    }
  }
  __device__ __forceinline__ void put_u32le(uint32_t v) { put_be32(bswap32(v)); }
  __device__ __forceinline__ void put_byte(uint32_t b) {
    total += 1;
    pend |= (b & 0xFFu) << (24 - 8 * pn);
    if (++pn == 4) {
      emit(pend);
      pend = 0;
      pn = 0;
    }
  }
  __device__ void put_bytes(const uint8_t* p, int64_t len) {
    int64_t i = 0;
    // bytes until the source is 4-aligned, then whole little-endian words
    while (i < len && (((uintptr_t)(p + i)) & 3u) != 0) put_byte(p[i++]);
    for (; i + 4 <= len; i += 4) put_be32(bswap32(__ldg(reinterpret_cast<const uint32_t*>(p + i))));
    for (; i < len; ++i) put_byte(p[i]);
  }
  // FIPS 180-4 padding, then lock-step compression of the buffered blocks.
  // Must be called by all 32 lanes (valid == false lanes only take part in the
  // lock-step loop bound).
  __device__ void finish(uint8_t* out, bool valid, uint32_t one) {
    int nb = 0;
    if (valid) {
      const uint64_t bits = total * 8;
      put_byte(0x80);
      while (pn != 0) put_byte(0);
      while ((nw & 15) != 14) emit(0);
      emit((uint32_t)(bits >> 32));
      emit((uint32_t)bits);
      nb = nw >> 4;
    }
    __syncwarp();
    const int nb_max = (int)__reduce_max_sync(0xFFFFFFFFu, (unsigned)nb);
    for (int b = 0; b < nb_max; ++b)
      if (b < nb) sha256_compress(h, buf + 16 * b, one);
    if (!valid) return;
    uint4* o4 = reinterpret_cast<uint4*>(out);
    o4[0] = make_uint4(bswap32(h[0]), bswap32(h[1]), bswap32(h[2]), bswap32(h[3]));
    o4[1] = make_uint4(bswap32(h[4]), bswap32(h[5]), bswap32(h[6]), bswap32(h[7]));
  }
  // The same digest into every peer rank's gathered array (fused all-gather).
  __device__ void broadcast(const dooly_digest_peers& pe, int64_t row) const {
    const uint4 a = make_uint4(bswap32(h[0]), bswap32(h[1]), bswap32(h[2]), bswap32(h[3]));
    const uint4 b = make_uint4(bswap32(h[4]), bswap32(h[5]), bswap32(h[6]), bswap32(h[7]));
    for (int p = 0; p < pe.n_peers; ++p) {
      uint4* o4 = reinterpret_cast<uint4*>(pe.digest[p] + row * 32);
      o4[0] = a;
      o4[1] = b;
    }
    if (pe.n_peers > 0) __threadfence_system();
  }
};

// LIST: hash only the records list[0 .. *count) (the representatives of the
// record grouping in dooly_dedup); each digest still lands at its record's row.
template <bool LIST>
__global__ void __launch_bounds__(SHA_THREADS, SHA_MINB) sha256_records_kernel(
    const uint32_t* __restrict__ words, const int64_t* __restrict__ rec_off, int64_t n,
    const uint8_t* __restrict__ op_bytes, const int64_t* __restrict__ op_off,
    const uint8_t* __restrict__ sym_bytes, const int64_t* __restrict__ sym_off,
    const uint8_t* __restrict__ attr_digests, uint8_t* __restrict__ out,
    const dooly_digest_peers pe, uint32_t one, const uint32_t* __restrict__ list,
    const uint32_t* __restrict__ count) {
  __shared__ uint32_t s_buf[SHA_THREADS * SHA_STRIDE];
  ShaStream st;
  const int64_t stride = (int64_t)gridDim.x * SHA_THREADS;
  const int64_t n_eff = LIST ? (int64_t)*count : n;
  for (int64_t base = (int64_t)blockIdx.x * SHA_THREADS; base < n_eff; base += stride) {
    const int64_t t = base + threadIdx.x;
    const bool valid = t < n_eff;
    const int64_t i = LIST ? (valid ? (int64_t)list[t] : 0) : t;
    st.init(s_buf + threadIdx.x * SHA_STRIDE);
    if (valid) {
    const uint32_t* r = words + rec_off[i];
    const uint32_t op = r[0], nd = r[1] & 0xFFFFu, ns = r[1] >> 16, attr = r[2];
    st.put_be32(0x73696766u);  // "sigf"
    st.put_be32(0x6d743d31u);  // "mt=1"
    const int64_t o0 = op_off[op], o1 = op_off[op + 1];
    st.put_u32le((uint32_t)(o1 - o0));
    st.put_bytes(op_bytes + o0, o1 - o0);
    st.put_u32le(nd);
    const uint32_t* dims = r + 4;
    for (uint32_t k = 0; k < 3 * nd; ++k) st.put_u32le(dims[k]);  // (pos, val_lo, val_hi)*
    st.put_u32le(ns);
    const uint32_t* syms = dims + 3 * nd;
    for (uint32_t k = 0; k < ns; ++k) {
      const int64_t s0 = sym_off[syms[k]], s1 = sym_off[syms[k] + 1];
      st.put_u32le((uint32_t)(s1 - s0));
      st.put_bytes(sym_bytes + s0, s1 - s0);
    }
    if (attr != 0xFFFFFFFFu) {
      const uint32_t* d = reinterpret_cast<const uint32_t*>(attr_digests + (int64_t)attr * 32);
      for (int k = 0; k < 8; ++k) st.put_be32(bswap32(d[k]));
    }
    }
    st.finish(out + (pe.row0 + i) * 32, valid, one);
    if (valid && pe.n_peers > 0) st.broadcast(pe, pe.row0 + i);
  }
}

__global__ void __launch_bounds__(SHA_THREADS) sha256_messages_kernel(
    const uint8_t* __restrict__ msgs, const int64_t* __restrict__ off, int64_t n,
    uint8_t* __restrict__ out, uint32_t one) {
  __shared__ uint32_t s_buf[SHA_THREADS * SHA_STRIDE];
  ShaStream st;
  for (int64_t base = (int64_t)blockIdx.x * SHA_THREADS; base < n;
       base += (int64_t)gridDim.x * SHA_THREADS) {
    const int64_t i = base + threadIdx.x;
    const bool valid = i < n;
    st.init(s_buf + threadIdx.x * SHA_STRIDE);
    if (valid) st.put_bytes(msgs + off[i], off[i + 1] - off[i]);
    st.finish(out + i * 32, valid, one);
  }
}

static int64_t sha_blocks(int64_t n, int n_sm) {
  int64_t blocks = (n + SHA_THREADS - 1) / SHA_THREADS;
  const int64_t cap = (int64_t)n_sm * 8;
  return blocks < cap ? blocks : cap;
}

cudaError_t launch_sha256_records(const uint32_t* words, const int64_t* rec_off, int64_t n,
                                  const uint8_t* op_bytes, const int64_t* op_off,
                                  const uint8_t* sym_bytes, const int64_t* sym_off,
                                  const uint8_t* attr_digests, uint8_t* out, cudaStream_t stream,
                                  int n_sm, int64_t* launches, const dooly_digest_peers* peers,
                                  const RecGroup* group) {
  if (n == 0) return cudaSuccess;
  *launches += 1;
  dooly_digest_peers pe{};
  if (peers) pe = *peers;
  if (group != nullptr)
    sha256_records_kernel<true><<<(unsigned)sha_blocks(n, n_sm), SHA_THREADS, 0, stream>>>(
        words, rec_off, n, op_bytes, op_off, sym_bytes, sym_off, attr_digests, out, pe, 1u,
        group->list, group->count);
  else
    sha256_records_kernel<false><<<(unsigned)sha_blocks(n, n_sm), SHA_THREADS, 0, stream>>>(
        words, rec_off, n, op_bytes, op_off, sym_bytes, sym_off, attr_digests, out, pe, 1u,
        nullptr, nullptr);
  return cudaGetLastError();
}

cudaError_t launch_sha256_messages(const uint8_t* msgs, const int64_t* off, int64_t n,
                                   uint8_t* out, cudaStream_t stream, int n_sm) {
  if (n == 0) return cudaSuccess;
  sha256_messages_kernel<<<(unsigned)sha_blocks(n, n_sm), SHA_THREADS, 0, stream>>>(msgs, off, n,
                                                                                     out, 1u);
  return cudaGetLastError();
}

}  // namespace dooly
