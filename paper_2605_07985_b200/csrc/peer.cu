// Peer-memory arrival counter for the fused compute + all-gather calls
// (dooly_fit_grid_bcast, dooly_sha256_records_bcast).  The producing kernel
// has already stored its rows into every rank's buffer over peer memory (CUDA
// IPC mappings; NVLink P2P stores on an NVSwitch box) and fenced them at
// system scope; here each rank adds 1 to every rank's counter and then waits
// until its own counter reaches the caller's target (world size x call
// number).  After the wait the gathered buffer is complete on this rank, in
// stream order — no host round trip and no NCCL call.
#include "common.cuh"

namespace dooly {

struct PeerFlags {
  int32_t n;
  uint32_t* f[DOOLY_MAX_PEERS];
};

__global__ void peer_signal_kernel(const PeerFlags pf, uint32_t* flag) {
  const int t = threadIdx.x;
  __threadfence_system();
  if (t < pf.n) {
    atomicAdd_system(pf.f[t], 1u);
  } else if (t == pf.n) {
    atomicAdd_system(flag, 1u);
  }
}

// Bounded wait: after ~20 s it raises *timed_out instead of hanging the GPU.
__global__ void peer_wait_kernel(const uint32_t* flag, uint32_t target, int32_t* timed_out) {
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if ((int32_t)(v - target) >= 0) break;
    uint64_t t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (t1 - t0 > 20ull * 1000000000ull) {
      *timed_out = 1;
      break;
    }
    __nanosleep(256);
  }
  __threadfence_system();
}

cudaError_t launch_peer_sync(int n_peers, uint32_t* const* peer_flags, uint32_t* flag,
                             uint32_t target, int32_t* timed_out, cudaStream_t stream,
                             int64_t* launches) {
  PeerFlags pf{};
  pf.n = n_peers;
  for (int p = 0; p < n_peers; ++p) pf.f[p] = peer_flags[p];
  peer_signal_kernel<<<1, 32, 0, stream>>>(pf, flag);
  peer_wait_kernel<<<1, 1, 0, stream>>>(flag, target, timed_out);
  *launches += 2;
  return cudaGetLastError();
}

}  // namespace dooly
