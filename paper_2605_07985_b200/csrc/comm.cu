// In-library NCCL communicator for the multi-GPU exchanges of the hot path
// (SURVEY §8(b) "dooly_comm_create / dooly_allgather", §8(e)): the one
// all-gather of fitted regressor rows, the dedup digest all-gather, and the
// owner-routed dedup's two all-to-alls.  The peer-memory fused forms
// (dooly_fit_grid_bcast, dooly_sha256_records_bcast) replace the all-gathers
// when every GPU pair has peer access; these are the NCCL forms beside them.
//
// Two ways to build a communicator:
//   * one process per GPU (the bench's torchrun layout): rank 0 calls
//     dooly_comm_unique_id, the 128 id bytes reach the other ranks out of band
//     (the caller's bootstrap), every rank calls dooly_comm_init_rank;
//   * one process driving several GPUs: dooly_comm_create (ncclCommInitAll).
// Calls are asynchronous on the caller's streams; errors return
// DOOLY_ERR_NCCL (message via dooly_comm_last_error).
#include <nccl.h>
#include <stdio.h>
#include <string.h>

#include <string>
#include <vector>

#include "common.cuh"

struct dooly_comm {
  std::vector<ncclComm_t> comms;  // one per local device
  std::vector<int> devs;
  int nranks = 0;                 // global ranks
  int rank0 = 0;                  // global rank of comms[0]
  std::string err;
};

static thread_local std::string g_comm_err;

static int nccl_fail(dooly_comm* c, ncclResult_t r, const char* what) {
  std::string m = std::string(what) + ": " + ncclGetErrorString(r);
  if (c) c->err = m;
  g_comm_err = m;
  return DOOLY_ERR_NCCL;
}

struct CommDeviceGuard {
  int prev = -1;
  explicit CommDeviceGuard(int d) {
    cudaGetDevice(&prev);
    if (d != prev) cudaSetDevice(d);
  }
  ~CommDeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

extern "C" {

int dooly_comm_unique_id(uint8_t* out) {
  if (!out) return DOOLY_ERR_INVALID_ARG;
  static_assert(sizeof(ncclUniqueId) == DOOLY_COMM_ID_BYTES, "NCCL unique id size");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(nullptr, r, "ncclGetUniqueId");
  memcpy(out, &id, sizeof(id));
  return DOOLY_OK;
}

int dooly_comm_init_rank(int device, const uint8_t* id, int nranks, int rank, dooly_comm** out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks || device < 0)
    return DOOLY_ERR_INVALID_ARG;
  dooly_comm* c = new dooly_comm();
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  CommDeviceGuard g(device);
  ncclComm_t comm;
  ncclResult_t r = ncclCommInitRank(&comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail(nullptr, r, "ncclCommInitRank");
  }
  c->comms.push_back(comm);
  c->devs.push_back(device);
  c->nranks = nranks;
  c->rank0 = rank;
  *out = c;
  return DOOLY_OK;
}

int dooly_comm_create(int ndev, const int* devs, dooly_comm** out) {
  if (ndev < 1 || !devs || !out) return DOOLY_ERR_INVALID_ARG;
  dooly_comm* c = new dooly_comm();
  c->comms.resize(ndev);
  c->devs.assign(devs, devs + ndev);
  ncclResult_t r = ncclCommInitAll(c->comms.data(), ndev, devs);
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail(nullptr, r, "ncclCommInitAll");
  }
  c->nranks = ndev;
  c->rank0 = 0;
  *out = c;
  return DOOLY_OK;
}

void dooly_comm_destroy(dooly_comm* c) {
  if (!c) return;
  for (size_t i = 0; i < c->comms.size(); ++i) {
    CommDeviceGuard g(c->devs[i]);
    ncclCommDestroy(c->comms[i]);
  }
  delete c;
}

const char* dooly_comm_last_error(const dooly_comm* c) {
  return c ? c->err.c_str() : g_comm_err.c_str();
}

int dooly_comm_size(const dooly_comm* c, int* nranks, int* rank0, int* n_local) {
  if (!c) return DOOLY_ERR_INVALID_ARG;
  if (nranks) *nranks = c->nranks;
  if (rank0) *rank0 = c->rank0;
  if (n_local) *n_local = (int)c->comms.size();
  return DOOLY_OK;
}

// In-place all-gather: bufs[i] is local device i's full buffer of nranks x
// bytes_per_rank; its own block sits at (rank0 + i) x bytes_per_rank.
int dooly_allgather(dooly_comm* c, void* const* bufs, size_t bytes_per_rank,
                    void* const* streams) {
  if (!c || !bufs || !streams) return DOOLY_ERR_INVALID_ARG;
  const int nl = (int)c->comms.size();
  for (int i = 0; i < nl; ++i)
    if (!bufs[i] && bytes_per_rank) return DOOLY_ERR_INVALID_ARG;
  if (bytes_per_rank == 0) return DOOLY_OK;
  ncclResult_t r = ncclGroupStart();
  if (r != ncclSuccess) return nccl_fail(c, r, "ncclGroupStart");
  for (int i = 0; i < nl; ++i) {
    char* b = static_cast<char*>(bufs[i]);
    r = ncclAllGather(b + (size_t)(c->rank0 + i) * bytes_per_rank, b, bytes_per_rank, ncclInt8,
                      c->comms[i], (cudaStream_t)streams[i]);
    if (r != ncclSuccess) {
      ncclGroupEnd();
      return nccl_fail(c, r, "ncclAllGather");
    }
  }
  r = ncclGroupEnd();
  if (r != ncclSuccess) return nccl_fail(c, r, "ncclGroupEnd");
  return DOOLY_OK;
}

// All-to-all with per-rank element counts (host arrays of nranks entries), for
// a communicator with one local device: send block p (the send_counts[p]
// elements after the first sum(send_counts[:p])) goes to rank p, recv block p
// comes from rank p.  Grouped ncclSend/ncclRecv.
int dooly_alltoallv(dooly_comm* c, const void* send, const int64_t* send_counts, void* recv,
                    const int64_t* recv_counts, size_t elem_bytes, void* stream) {
  if (!c || !send_counts || !recv_counts || elem_bytes == 0 || c->comms.size() != 1)
    return DOOLY_ERR_INVALID_ARG;
  const char* s = static_cast<const char*>(send);
  char* d = static_cast<char*>(recv);
  size_t so = 0, ro = 0;
  ncclResult_t r = ncclGroupStart();
  if (r != ncclSuccess) return nccl_fail(c, r, "ncclGroupStart");
  for (int p = 0; p < c->nranks; ++p) {
    const size_t sb = (size_t)send_counts[p] * elem_bytes, rb = (size_t)recv_counts[p] * elem_bytes;
    if (sb) r = ncclSend(s + so, sb, ncclInt8, p, c->comms[0], (cudaStream_t)stream);
    if (r == ncclSuccess && rb) r = ncclRecv(d + ro, rb, ncclInt8, p, c->comms[0], (cudaStream_t)stream);
    if (r != ncclSuccess) {
      ncclGroupEnd();
      return nccl_fail(c, r, "ncclSend/ncclRecv");
    }
    so += sb;
    ro += rb;
  }
  r = ncclGroupEnd();
  if (r != ncclSuccess) return nccl_fail(c, r, "ncclGroupEnd");
  return DOOLY_OK;
}

}  // extern "C"
