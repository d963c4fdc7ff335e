// FP64 throughput probe on this B200: vector DFMA vs warp-level DMMA
// (mma.sync m8n8k4 / m16n8k4 / m16n8k8 / m16n8k16 .f64).  Built by tools/fp64_probe.py.
#include <cuda_runtime.h>
#include <stdint.h>

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 1.2345) out[0] = s;
}

template <int CHAINS>
__global__ void dmma884_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = threadIdx.x * 2e-3;
  double c0[CHAINS], c1[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) c0[c] = c1[c] = c;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c0[c]), "+d"(c1[c])
                   : "d"(a), "d"(b));
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += c0[c] + c1[c];
  if (s == 1.2345) out[0] = s;
}

template <int CHAINS>
__global__ void dmma1684_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 * 3, b = threadIdx.x * 2e-3;
  double c[CHAINS][4];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k)
#pragma unroll
    for (int j = 0; j < 4; ++j) c[k][j] = k + j;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < CHAINS; ++k)
      asm volatile(
          "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
          "{%0,%1,%2,%3};"
          : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
          : "d"(a0), "d"(a1), "d"(b));
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k)
#pragma unroll
    for (int j = 0; j < 4; ++j) s += c[k][j];
  if (s == 1.2345) out[0] = s;
}

template <int CHAINS>
__global__ void dmma16816_kernel(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
#pragma unroll
  for (int j = 0; j < 4; ++j) b[j] = threadIdx.x * 2e-3 + j;
  double c[CHAINS][4];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k)
#pragma unroll
    for (int j = 0; j < 4; ++j) c[k][j] = k + j;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < CHAINS; ++k)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
          "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
          : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]),
            "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k)
#pragma unroll
    for (int j = 0; j < 4; ++j) s += c[k][j];
  if (s == 1.2345) out[0] = s;
}

template <int CHAINS>
__global__ void mixed_kernel(double* out, int iters, double fa, double fb) {
  double a = threadIdx.x * 1e-3, b = threadIdx.x * 2e-3;
  double c0[CHAINS], c1[CHAINS], v[8];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) c0[c] = c1[c] = c;
#pragma unroll
  for (int c = 0; c < 8; ++c) v[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c0[c]), "+d"(c1[c])
                   : "d"(a), "d"(b));
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) v[c] = fma(v[c], fa, fb);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += c0[c] + c1[c];
#pragma unroll
  for (int c = 0; c < 8; ++c) s += v[c];
  if (s == 1.2345) out[0] = s;
}

// returns FMA operations per launch (for FLOP/s = 2 * fma / time)
extern "C" double probe_fp64(int which, int blocks, int threads, int iters, double* out,
                             void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const double warps = (double)blocks * threads / 32.0;
  switch (which) {
    case 0:
      dfma_kernel<8><<<blocks, threads, 0, s>>>(out, iters, 1.0000001, 1e-9);
      return warps * 32 * 8.0 * iters;
    case 1:
      dmma884_kernel<4><<<blocks, threads, 0, s>>>(out, iters);
      return warps * 4 * 256.0 * iters;
    case 2:
      dmma1684_kernel<4><<<blocks, threads, 0, s>>>(out, iters);
      return warps * 4 * 512.0 * iters;
    case 3:
      dmma16816_kernel<4><<<blocks, threads, 0, s>>>(out, iters);
      return warps * 4 * 2048.0 * iters;
    case 4:  // 4 DMMA (1024 FMA) + 32 DFMA per lane (1024 FMA) per warp-iteration
      mixed_kernel<4><<<blocks, threads, 0, s>>>(out, iters, 1.0000001, 1e-9);
      return warps * (4 * 256.0 + 32 * 32.0) * iters;
  }
  return 0;
}
