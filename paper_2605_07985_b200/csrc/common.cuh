// Shared device helpers for libdooly_b200 (sm_100a).
//
// The regression evaluation here is THE parity contract for predictions:
// features are scaled with one correctly-rounded multiply, every monomial
// and every term is a separate __dmul_rn / __dadd_rn (no FMA contraction),
// in the fixed order of SURVEY.md App. A.7 / A.11.  oracle/sim.py performs
// the identical sequence with numpy float64 (which never contracts), so given
// the same table row the two sides agree bit-for-bit.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/dooly_b200.h"

#define DOOLY_CLAMP_FLOOR 1e-7  // SPEC.md:569 / :574

namespace dooly {

static_assert(sizeof(dooly_affine_row) == 32, "affine row must be one 32-B sector");
static_assert(sizeof(dooly_attn_row) == 128, "attention row must be one 128-B line");

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }

// Non-caching streaming loads for data read exactly once.
__device__ __forceinline__ uint4 ld_stream_u4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ld_stream_u32(const void* p) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream_f64x2(double* p, double a, double b) {
  asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(a), "d"(b)
               : "memory");
}

// ---- rows ---------------------------------------------------------------
struct AffineRow {  // mirrors dooly_affine_row; loaded as two 16-B vectors
  double c0, c1, inv;
  uint32_t lo, hi;
};
struct AttnRow {
  double c[10];
  double inv[3];
  uint32_t lo[3], hi[3];
};

__device__ __forceinline__ AffineRow load_affine(const dooly_affine_row* t, uint32_t s) {
  const double2* p = reinterpret_cast<const double2*>(t + s);
  double2 a = __ldg(p);
  double2 b = __ldg(p + 1);
  AffineRow r;
  r.c0 = a.x;
  r.c1 = a.y;
  r.inv = b.x;
  uint2 box = *reinterpret_cast<const uint2*>(&b.y);
  r.lo = box.x;
  r.hi = box.y;
  return r;
}

__device__ __forceinline__ AttnRow load_attn(const dooly_attn_row* t, uint32_t s) {
  const double2* p = reinterpret_cast<const double2*>(t + s);
  AttnRow r;
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    double2 v = __ldg(p + i);
    r.c[2 * i] = v.x;
    r.c[2 * i + 1] = v.y;
  }
  double2 v5 = __ldg(p + 5);
  double2 v6 = __ldg(p + 6);
  uint4 box = __ldg(reinterpret_cast<const uint4*>(p + 7));
  r.inv[0] = v5.x;
  r.inv[1] = v5.y;
  r.inv[2] = v6.x;
  uint2 b0 = *reinterpret_cast<const uint2*>(&v6.y);
  r.lo[0] = b0.x;
  r.lo[1] = b0.y;
  r.lo[2] = box.x;
  r.hi[0] = box.y;
  r.hi[1] = box.z;
  r.hi[2] = box.w;
  return r;
}

// ---- evaluation (parity contract) ----------------------------------------
__device__ __forceinline__ double eval_affine(const AffineRow& r, uint32_t x) {
  double f = mul((double)x, r.inv);
  return add(r.c0, mul(r.c1, f));
}

__device__ __forceinline__ double eval_attn(const AttnRow& r, uint32_t x0, uint32_t x1,
                                            uint32_t x2) {
  double f1 = mul((double)x0, r.inv[0]);
  double f2 = mul((double)x1, r.inv[1]);
  double f3 = mul((double)x2, r.inv[2]);
  double p = r.c[0];
  p = add(p, mul(r.c[1], f1));
  p = add(p, mul(r.c[2], f2));
  p = add(p, mul(r.c[3], f3));
  p = add(p, mul(r.c[4], mul(f1, f1)));
  p = add(p, mul(r.c[5], mul(f2, f2)));
  p = add(p, mul(r.c[6], mul(f3, f3)));
  p = add(p, mul(r.c[7], mul(f1, f2)));
  p = add(p, mul(r.c[8], mul(f1, f3)));
  p = add(p, mul(r.c[9], mul(f2, f3)));
  return p;
}

// ---- packed serving rows (DOOLY_KIND_ATTN_PACKED; parity contract) --------
// The 96-B serving row carries the coefficients FOLDED into raw-feature
// space (inv = RN(1/hi), 1 if hi == 0), grouped by feature: sector k holds
// everything that multiplies feature k first,
//   a_k = c_{1+k} * inv_k,  b_k = (c_{4+k} * inv_k) * inv_k,
//   d_0 = (c7 * inv_0) * inv_1,  d_1 = (c9 * inv_1) * inv_2,  d_2 = (c8 * inv_0) * inv_2,
// as words {e_k, a_k, b_k, d_k} with e_0 = c0, e_1 = lo_bits, e_2 = hi_bits.
// The value is the per-feature 3-way tree over raw features
//   s_k = ((e'_k + a_k x_k) + b_k (x_k x_k)) + d_k (x_k x_{k+1 mod 3}),
//   e'_0 = c0, e'_1 = e'_2 = 0,        p = (s_0 + s_1) + s_2,
// so lane k of a 3-lane group evaluates s_k from its own 32-B sector and its
// own two feature planes (predict.cu).  oracle/sim.py pack_attn /
// eval_folded perform the identical operations.
__device__ __forceinline__ void fold_row96(const double* c, const double* inv, uint64_t lo_bits,
                                           uint64_t hi_bits, double* w) {
  w[0] = c[0];
  w[1] = mul(c[1], inv[0]);
  w[2] = mul(mul(c[4], inv[0]), inv[0]);
  w[3] = mul(mul(c[7], inv[0]), inv[1]);
  w[4] = __longlong_as_double((long long)lo_bits);
  w[5] = mul(c[2], inv[1]);
  w[6] = mul(mul(c[5], inv[1]), inv[1]);
  w[7] = mul(mul(c[9], inv[1]), inv[2]);
  w[8] = __longlong_as_double((long long)hi_bits);
  w[9] = mul(c[3], inv[2]);
  w[10] = mul(mul(c[6], inv[2]), inv[2]);
  w[11] = mul(mul(c[8], inv[0]), inv[2]);
}

// s_k of the tree (e = e'_k, x = x_k, y = x_{k+1})
__device__ __forceinline__ double sector_sum(double e, double a, double b, double d, double x,
                                             double y) {
  return add(add(add(e, mul(a, x)), mul(b, mul(x, x))), mul(d, mul(x, y)));
}

__device__ __forceinline__ double eval_row96(const double* w, uint32_t x0, uint32_t x1,
                                             uint32_t x2) {
  const double a = (double)x0, b = (double)x1, c = (double)x2;
  const double s0 = sector_sum(w[0], w[1], w[2], w[3], a, b);
  const double s1 = sector_sum(0.0, w[5], w[6], w[7], b, c);
  const double s2 = sector_sum(0.0, w[9], w[10], w[11], c, a);
  return add(add(s0, s1), s2);
}

__device__ __forceinline__ bool affine_valid(const AffineRow& r) { return r.lo <= r.hi; }
__device__ __forceinline__ bool attn_valid(const AttnRow& r) { return r.lo[0] <= r.hi[0]; }

__device__ __forceinline__ double clamp_floor(double p, bool& clamped) {
  clamped = p < DOOLY_CLAMP_FLOOR;
  return clamped ? DOOLY_CLAMP_FLOOR : p;
}

__device__ __forceinline__ double nan64() { return __longlong_as_double(0x7ff8000000000000ll); }

// Record grouping ahead of SHA-256 (dedup.cu): per record its representative
// (a record with identical packed content), the representatives' list and count.
struct RecGroup {
  uint32_t* rep;
  uint32_t* list;
  uint32_t* count;
};

}  // namespace dooly
