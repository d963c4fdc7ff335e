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

__device__ __forceinline__ bool affine_valid(const AffineRow& r) { return r.lo <= r.hi; }
__device__ __forceinline__ bool attn_valid(const AttnRow& r) { return r.lo[0] <= r.hi[0]; }

__device__ __forceinline__ double clamp_floor(double p, bool& clamped) {
  clamped = p < DOOLY_CLAMP_FLOOR;
  return clamped ? DOOLY_CLAMP_FLOOR : p;
}

__device__ __forceinline__ double nan64() { return __longlong_as_double(0x7ff8000000000000ll); }

}  // namespace dooly
