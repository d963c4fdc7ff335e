// Peer-memory counters for the fused compute + all-gather calls
// (dooly_fit_grid_bcast, dooly_sha256_records_bcast).  Two handshakes per
// call: "ready" before the producing kernel (every rank has stopped reading
// the previous call's buffers: no write-after-read), "arrived" after it (the
// kernel has stored its rows into every rank's buffer over peer memory — CUDA
// IPC mappings; NVLink P2P stores on an NVSwitch box — and fenced them at
// system scope).  After the second wait the gathered buffer is complete on
// this rank, in stream order — no host round trip and no NCCL call.
#include "common.cuh"

namespace dooly {

struct PeerFlags {
  int32_t n;
  uint32_t* f[DOOLY_MAX_PEERS];
};

// slot 0: arrivals (my rows are in every rank's buffer); slot 1: ready (I no
// longer read the previous call's contents of my buffers, peers may overwrite).
__global__ void peer_signal_kernel(const PeerFlags pf, uint32_t* flag, int slot) {
  const int t = threadIdx.x;
  __threadfence_system();
  if (t < pf.n) {
    atomicAdd_system(pf.f[t] + slot, 1u);
  } else if (t == pf.n) {
    atomicAdd_system(flag + slot, 1u);
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

// Handshake on counter `slot` of every rank's flag buffer (flag[0] arrivals,
// flag[1] ready): add 1 to every rank's counter, then wait on the stream
// until this rank's counter reaches `target` (world size x call number).
//   * before the producing kernel, slot 1 ("ready"): every rank has reached
//     this call in its stream, so nothing it enqueued earlier still reads the
//     buffers this call overwrites (the consumer-done barrier: no
//     write-after-read across ranks);
//   * after it, slot 0 ("arrived"): every rank's rows are in every buffer.
cudaError_t launch_peer_sync(int n_peers, uint32_t* const* peer_flags, uint32_t* flag,
                             uint32_t target, int32_t* timed_out, cudaStream_t stream,
                             int64_t* launches, int slot) {
  PeerFlags pf{};
  pf.n = n_peers;
  for (int p = 0; p < n_peers; ++p) pf.f[p] = peer_flags[p];
  peer_signal_kernel<<<1, 32, 0, stream>>>(pf, flag, slot);
  peer_wait_kernel<<<1, 1, 0, stream>>>(flag + slot, target, timed_out);
  *launches += 2;
  return cudaGetLastError();
}

cudaError_t enable_peer_access(int device, int peer) {
  int cur = 0;
  cudaError_t e = cudaGetDevice(&cur);
  if (e != cudaSuccess) return e;
  if (peer == device) return cudaSuccess;
  int can = 0;
  e = cudaDeviceCanAccessPeer(&can, device, peer);
  if (e != cudaSuccess) return e;
  if (!can) return cudaErrorPeerAccessUnsupported;
  e = cudaSetDevice(device);
  if (e != cudaSuccess) return e;
  e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    (void)cudaGetLastError();  // clear the sticky-free error state
    e = cudaSuccess;
  }
  cudaSetDevice(cur);
  return e;
}

}  // namespace dooly
