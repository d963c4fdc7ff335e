// extern "C" boundary of libdooly_b200 (include/dooly_b200.h).
// Validates arguments, selects the kernel, launches on the caller's stream,
// and records errors for dooly_last_error().  No allocation, no host sync.
#include <stdio.h>
#include <string.h>

#include <string>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"

namespace dooly {
cudaError_t launch_predict(int kind, const void* table, int64_t n_sig, const uint32_t* sig,
                           const uint32_t* x, int64_t n_q, double* out, uint32_t* flags,
                           int64_t* err_first, cudaStream_t stream, int n_sm);
cudaError_t launch_fit(int kind, const uint32_t* x, int64_t n_pts, const double* y,
                       const int64_t* off, int64_t n_sig, void* table, double* fit_err,
                       uint8_t* status, void* ws, cudaStream_t stream, int n_sm,
                       int64_t* launches);
size_t fit_workspace_size(int kind, int64_t n_sig);
size_t fit_grid_workspace_size(int kind, int64_t n_pts);
cudaError_t launch_fit_grid(int kind, const uint32_t* x, int64_t n_pts, const double* y,
                            int64_t n_sig, void* table, double* fit_err, uint8_t* status,
                            const dooly_grid_peers* peers, void* ws, cudaStream_t stream,
                            int n_sm, int64_t* launches, void* packed = nullptr);
cudaError_t launch_attn_pack(const void* table, int64_t n_sig, void* packed, cudaStream_t stream,
                             int n_sm, int64_t* launches);
cudaError_t launch_sha256_records(const uint32_t* words, const int64_t* rec_off, int64_t n,
                                  const uint8_t* op_bytes, const int64_t* op_off,
                                  const uint8_t* sym_bytes, const int64_t* sym_off,
                                  const uint8_t* attr_digests, uint8_t* out, cudaStream_t stream,
                                  int n_sm, int64_t* launches,
                                  const dooly_digest_peers* peers = nullptr,
                                  const RecGroup* group = nullptr);
RecGroup rec_group_carve(void* ws, int64_t n, int64_t n_db);
cudaError_t launch_rec_group(const uint32_t* words, const int64_t* rec_off, int64_t n, void* ws,
                             int64_t n_db, cudaStream_t stream, int n_sm, int64_t* launches);
cudaError_t launch_digest_copy(const uint32_t* rep, int64_t n, uint8_t* digests,
                               cudaStream_t stream, int n_sm, int64_t* launches);
cudaError_t launch_peer_sync(int n_peers, uint32_t* const* peer_flags, uint32_t* flag,
                             uint32_t target, int32_t* timed_out, cudaStream_t stream,
                             int64_t* launches, int slot);
cudaError_t enable_peer_access(int device, int peer);
cudaError_t launch_dedup_firsts(int64_t n, int64_t n_db, const int64_t* gidx, int64_t* out_firsts,
                                void* ws, cudaStream_t stream, int n_sm, int64_t* launches);
size_t route_workspace_size(int64_t n, int world);
cudaError_t launch_route_plan(const uint8_t* dig, int64_t n, int world, int64_t gidx0,
                              int64_t* perm, int64_t* counts, uint8_t* out_dig, int64_t* out_gidx,
                              void* ws, cudaStream_t stream, int64_t* launches);
cudaError_t launch_route_reply(const int64_t* gidx, const int64_t* first, const uint8_t* is_new,
                               const uint8_t* in_db, int64_t m, const int64_t* all_firsts,
                               int64_t per, int world, int64_t* rows, cudaStream_t stream,
                               int n_sm, int64_t* launches);
cudaError_t launch_route_finish(const int64_t* rows, const int64_t* perm, int64_t n,
                                int64_t* out_first, uint32_t* out_uid, uint8_t* out_is_new,
                                uint8_t* out_in_db, cudaStream_t stream, int n_sm,
                                int64_t* launches);
cudaError_t launch_sha256_messages(const uint8_t* msgs, const int64_t* off, int64_t n,
                                   uint8_t* out, cudaStream_t stream, int n_sm);
size_t dedup_workspace_size(int64_t n, int64_t n_db);
cudaError_t launch_dedup(const uint8_t* digests, int64_t n, const uint8_t* db, int64_t n_db,
                         int64_t* out_first, uint32_t* out_uid, uint8_t* out_is_new,
                         uint8_t* out_in_db, int64_t* out_n_unique, void* ws, size_t ws_bytes,
                         cudaStream_t stream, int n_sm, int64_t* launches,
                         const uint32_t* grp = nullptr);
cudaError_t launch_iter_eval(const dooly_oplist* ops, const void* aff, int64_t n_aff,
                             const void* attn, int64_t n_attn, const uint32_t* it_feat,
                             int64_t n_it, double* it_lat, int64_t* err_first,
                             cudaStream_t stream, int n_sm);
size_t sim_workspace_size(const dooly_sched* cfg, int64_t n_req, int64_t n_shards);
cudaError_t launch_sim_eval(const double* it_lat, const double* it_start, const int64_t* it_off,
                            int64_t n_shards, int64_t n_it, double* clock, const double* arrival,
                            const uint32_t* first_it, const uint32_t* last_it,
                            const uint32_t* out_tok, int64_t n_req, double* ttft, double* tpot,
                            int64_t* err_first, cudaStream_t stream, int n_sm,
                            int64_t* launches);
cudaError_t launch_profile_fit(int kind, const dooly_sweep_desc* descs, int64_t n_sig,
                               const dooly_sweep_grid* grid, void* table, double* fit_err,
                               uint8_t* status, uint32_t* out_x, double* out_y,
                               const int64_t* out_off, int64_t out_n, cudaStream_t stream,
                               int n_sm);
cudaError_t launch_sim(const dooly_oplist* ops, const dooly_sched* cfg, const void* aff,
                       int64_t n_aff, const void* attn, int64_t n_attn, const double* arrival,
                       const uint32_t* prompt, const uint32_t* output, const uint32_t* cached,
                       const int64_t* shard_off, int64_t n_shards, double* ttft, double* tpot,
                       int64_t* n_iter, double* final_clock, int32_t* shard_status,
                       uint32_t* it_log_feat, double* it_log_lat, int64_t it_log_cap, void* ws,
                       size_t ws_bytes, cudaStream_t stream, int n_sm);
}  // namespace dooly

struct dooly_ctx {
  int device = 0;
  int n_sm = 148;
  int64_t launches = 0;
  std::string err;
};

namespace {

int fail(dooly_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

int check_cuda(dooly_ctx* ctx, cudaError_t e, const char* where) {
  if (e == cudaSuccess) return DOOLY_OK;
  return fail(ctx, DOOLY_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// Guard: every call runs on the ctx's device.
// Device guard of every launching entry point, also an NVTX range named after
// the entry point (SURVEY §5 tracing: host-side ranges nsys / ncu --nvtx can
// filter on; no-ops without a tool attached).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev, const char* range = nullptr) {
    if (range) nvtxRangePushA(range);
    pushed = range != nullptr;
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    if (pushed) nvtxRangePop();
  }
  bool pushed = false;
};

}  // namespace

extern "C" {

int dooly_version(void) { return DOOLY_ABI_VERSION; }

int dooly_ctx_create(int device, dooly_ctx** out) {
  if (out == nullptr) return DOOLY_ERR_INVALID_ARG;
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || device < 0 || device >= n) return DOOLY_ERR_CUDA;
  dooly_ctx* c = new dooly_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->n_sm, cudaDevAttrMultiProcessorCount, device);
  *out = c;
  return DOOLY_OK;
}

void dooly_ctx_destroy(dooly_ctx* ctx) { delete ctx; }

const char* dooly_last_error(const dooly_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

int64_t dooly_launch_count(const dooly_ctx* ctx) { return ctx ? ctx->launches : 0; }

int dooly_predict(dooly_ctx* ctx, int kind, const void* table, int64_t n_sig,
                  const uint32_t* sig, const uint32_t* x, int64_t n_q, double* out,
                  uint32_t* flag_bits, int64_t* err_first, void* stream) {
  if (!ctx) return DOOLY_ERR_INVALID_ARG;
  if (kind != DOOLY_KIND_AFFINE && kind != DOOLY_KIND_ATTN && kind != DOOLY_KIND_ATTN_PACKED)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "predict: unknown kind");
  if (kind == DOOLY_KIND_ATTN_PACKED && !table)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "predict: packed table needs its header");
  if (n_q < 0 || n_sig < 0) return fail(ctx, DOOLY_ERR_INVALID_ARG, "predict: negative size");
  if (n_q > 0 && (!table && n_sig > 0 || !sig || !x || !out))
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "predict: null pointer");
  if ((uintptr_t)table % 32 != 0)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "predict: table must be 32-byte aligned");
  DeviceGuard g(ctx->device, __func__);
  if (n_q > 0) ctx->launches += 1;
  return check_cuda(ctx,
                    dooly::launch_predict(kind, table, n_sig, sig, x, n_q, out, flag_bits,
                                          err_first, (cudaStream_t)stream, ctx->n_sm),
                    "predict");
}

size_t dooly_attn_pack_bytes(int64_t n_sig) {
  return n_sig < 0 ? 0 : (size_t)(n_sig + 1) * sizeof(dooly_attn_row96);
}

int dooly_attn_pack(dooly_ctx* ctx, const void* table, int64_t n_sig, void* packed,
                    void* stream) {
  if (!ctx) return DOOLY_ERR_INVALID_ARG;
  if (n_sig < 0) return fail(ctx, DOOLY_ERR_INVALID_ARG, "attn_pack: negative size");
  if (!packed || (n_sig > 0 && !table))
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "attn_pack: null pointer");
  if ((uintptr_t)packed % 32 != 0 || (uintptr_t)table % 16 != 0)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "attn_pack: packed must be 32-B, table 16-B aligned");
  if (n_sig > 0xFFFFFFFFll)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "attn_pack: more than 2^32 rows");
  DeviceGuard g(ctx->device, __func__);
  return check_cuda(ctx,
                    dooly::launch_attn_pack(table, n_sig, packed, (cudaStream_t)stream,
                                            ctx->n_sm, &ctx->launches),
                    "attn_pack");
}

size_t dooly_fit_workspace_size(int kind, int64_t n_sig) {
  return dooly::fit_workspace_size(kind, n_sig);
}

int dooly_fit(dooly_ctx* ctx, int kind, const uint32_t* x, int64_t n_pts, const double* y,
              const int64_t* pt_off, int64_t n_sig, void* table, double* fit_err,
              uint8_t* status, void* workspace, size_t workspace_bytes, void* stream) {
  if (!ctx) return DOOLY_ERR_INVALID_ARG;
  if (kind != DOOLY_KIND_AFFINE && kind != DOOLY_KIND_ATTN)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "fit: unknown kind");
  if (n_sig < 0 || n_pts < 0) return fail(ctx, DOOLY_ERR_INVALID_ARG, "fit: negative size");
  if (n_sig > 0 && (!pt_off || !table || !fit_err || !status || (n_pts > 0 && (!x || !y))))
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "fit: null pointer");
  if (workspace != nullptr &&
      (workspace_bytes < dooly::fit_workspace_size(kind, n_sig) || (uintptr_t)workspace % 256))
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "fit: workspace too small or misaligned");
  DeviceGuard g(ctx->device, __func__);
  return check_cuda(ctx,
                    dooly::launch_fit(kind, x, n_pts, y, pt_off, n_sig, table, fit_err, status,
                                      workspace, (cudaStream_t)stream, ctx->n_sm,
                                      &ctx->launches),
                    "fit");
}

size_t dooly_fit_grid_workspace_size(int kind, int64_t n_pts) {
  return dooly::fit_grid_workspace_size(kind, n_pts);
}

int dooly_fit_grid(dooly_ctx* ctx, int kind, const uint32_t* x, int64_t n_pts, const double* y,
                   int64_t n_sig, void* table, double* fit_err, uint8_t* status, void* workspace,
                   size_t workspace_bytes, void* stream) {
  if (!ctx) return DOOLY_ERR_INVALID_ARG;
  if (kind != DOOLY_KIND_AFFINE && kind != DOOLY_KIND_ATTN)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "fit_grid: unknown kind");
  if (n_sig < 0 || n_pts < 0) return fail(ctx, DOOLY_ERR_INVALID_ARG, "fit_grid: negative size");
  if (!workspace || workspace_bytes < dooly::fit_grid_workspace_size(kind, n_pts) ||
      (uintptr_t)workspace % 16)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "fit_grid: workspace too small or misaligned");
  if ((n_pts > 0 && !x) || (n_sig > 0 && (!table || !fit_err || !status || (n_pts > 0 && !y))))
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "fit_grid: null pointer");
  if ((uintptr_t)table % 16)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "fit_grid: table must be 16-byte aligned");
  DeviceGuard g(ctx->device, __func__);
  return check_cuda(ctx,
                    dooly::launch_fit_grid(kind, x, n_pts, y, n_sig, table, fit_err, status,
                                           nullptr, workspace, (cudaStream_t)stream, ctx->n_sm,
                                           &ctx->launches),
                    "fit_grid");
}

int dooly_fit_grid_packed(dooly_ctx* ctx, const uint32_t* x, int64_t n_pts, const double* y,
                          int64_t n_sig, void* table, double* fit_err, uint8_t* status,
                          void* packed, void* workspace, size_t workspace_bytes, void* stream) {
  if (!ctx) return DOOLY_ERR_INVALID_ARG;
  const int kind = DOOLY_KIND_ATTN;
  if (n_sig < 0 || n_pts < 0)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "fit_grid_packed: negative size");
  if (!workspace || workspace_bytes < dooly::fit_grid_workspace_size(kind, n_pts) ||
      (uintptr_t)workspace % 16)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "fit_grid_packed: workspace too small or misaligned");
  if (!packed || (n_pts > 0 && !x) ||
      (n_sig > 0 && (!table || !fit_err || !status || (n_pts > 0 && !y))))
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "fit_grid_packed: null pointer");
  if ((uintptr_t)table % 16 || (uintptr_t)packed % 16)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "fit_grid_packed: table and packed must be 16-byte aligned");
  DeviceGuard g(ctx->device, __func__);
  return check_cuda(ctx,
                    dooly::launch_fit_grid(kind, x, n_pts, y, n_sig, table, fit_err, status,
                                           nullptr, workspace, (cudaStream_t)stream, ctx->n_sm,
                                           &ctx->launches, packed),
                    "fit_grid_packed");
}

int dooly_fit_grid_bcast(dooly_ctx* ctx, int kind, const uint32_t* x, int64_t n_pts,
                         const double* y, int64_t n_sig, void* table, double* fit_err,
                         uint8_t* status, const dooly_grid_peers* peers, uint32_t* flag,
                         uint32_t target, int32_t* timed_out, void* workspace,
                         size_t workspace_bytes, void* stream) {
  if (!ctx) return DOOLY_ERR_INVALID_ARG;
  if (!peers || peers->n_peers < 0 || peers->n_peers > DOOLY_MAX_PEERS || peers->row0 < 0 ||
      !flag || !timed_out)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "fit_grid_bcast: bad peer set");
  for (int p = 0; p < peers->n_peers; ++p)
    if (!peers->table[p] || !peers->fit_err[p] || !peers->status[p] || !peers->flag[p] ||
        (uintptr_t)peers->table[p] % 16)
      return fail(ctx, DOOLY_ERR_INVALID_ARG, "fit_grid_bcast: null or misaligned peer buffer");
  if (kind != DOOLY_KIND_AFFINE && kind != DOOLY_KIND_ATTN)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "fit_grid_bcast: unknown kind");
  if (n_sig < 0 || n_pts < 0) return fail(ctx, DOOLY_ERR_INVALID_ARG, "fit_grid_bcast: negative size");
  if (!workspace || workspace_bytes < dooly::fit_grid_workspace_size(kind, n_pts) ||
      (uintptr_t)workspace % 16)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "fit_grid_bcast: workspace too small or misaligned");
  if ((n_pts > 0 && !x) || (n_sig > 0 && (!table || !fit_err || !status || (n_pts > 0 && !y))))
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "fit_grid_bcast: null pointer");
  if ((uintptr_t)table % 16)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "fit_grid_bcast: table must be 16-byte aligned");
  DeviceGuard g(ctx->device, __func__);
  cudaError_t e = dooly::launch_peer_sync(peers->n_peers, peers->flag, flag, target, timed_out,
                                          (cudaStream_t)stream, &ctx->launches, 1);
  if (e == cudaSuccess)
    e = dooly::launch_fit_grid(kind, x, n_pts, y, n_sig, table, fit_err, status, peers,
                               workspace, (cudaStream_t)stream, ctx->n_sm, &ctx->launches);
  if (e == cudaSuccess)
    e = dooly::launch_peer_sync(peers->n_peers, peers->flag, flag, target, timed_out,
                                (cudaStream_t)stream, &ctx->launches, 0);
  return check_cuda(ctx, e, "fit_grid_bcast");
}

int dooly_sha256_records(dooly_ctx* ctx, const uint32_t* words, const int64_t* rec_off,
                         int64_t n, const uint8_t* op_bytes, const int64_t* op_off,
                         int64_t n_ops, const uint8_t* sym_bytes, const int64_t* sym_off,
                         int64_t n_sym, const uint8_t* attr_digests, int64_t n_attr,
                         uint8_t* out_digest, void* stream) {
  (void)n_ops;
  (void)n_sym;
  (void)n_attr;
  if (!ctx) return DOOLY_ERR_INVALID_ARG;
  if (n < 0) return fail(ctx, DOOLY_ERR_INVALID_ARG, "sha256_records: negative size");
  if (n > 0 && (!words || !rec_off || !op_bytes || !op_off || !out_digest))
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "sha256_records: null pointer");
  DeviceGuard g(ctx->device, __func__);
  return check_cuda(ctx,
                    dooly::launch_sha256_records(words, rec_off, n, op_bytes, op_off, sym_bytes,
                                                 sym_off, attr_digests, out_digest,
                                                 (cudaStream_t)stream, ctx->n_sm,
                                                 &ctx->launches),
                    "sha256_records");
}

int dooly_sha256_records_bcast(dooly_ctx* ctx, const uint32_t* words, const int64_t* rec_off,
                               int64_t n, const uint8_t* op_bytes, const int64_t* op_off,
                               int64_t n_ops, const uint8_t* sym_bytes, const int64_t* sym_off,
                               int64_t n_sym, const uint8_t* attr_digests, int64_t n_attr,
                               uint8_t* out_digest, const dooly_digest_peers* peers,
                               uint32_t* flag, uint32_t target, int32_t* timed_out,
                               void* stream) {
  (void)n_ops;
  (void)n_sym;
  (void)n_attr;
  if (!ctx) return DOOLY_ERR_INVALID_ARG;
  if (n < 0) return fail(ctx, DOOLY_ERR_INVALID_ARG, "sha256_records_bcast: negative size");
  if (n > 0 && (!words || !rec_off || !op_bytes || !op_off || !out_digest))
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "sha256_records_bcast: null pointer");
  if (!peers || peers->n_peers < 0 || peers->n_peers > DOOLY_MAX_PEERS || peers->row0 < 0 ||
      !flag || !timed_out)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "sha256_records_bcast: bad peer set");
  for (int p = 0; p < peers->n_peers; ++p)
    if (!peers->digest[p] || !peers->flag[p] || (uintptr_t)peers->digest[p] % 16)
      return fail(ctx, DOOLY_ERR_INVALID_ARG,
                  "sha256_records_bcast: null or misaligned peer buffer");
  if ((uintptr_t)out_digest % 16)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "sha256_records_bcast: digests must be 16-B aligned");
  DeviceGuard g(ctx->device, __func__);
  cudaError_t e = dooly::launch_peer_sync(peers->n_peers, peers->flag, flag, target, timed_out,
                                          (cudaStream_t)stream, &ctx->launches, 1);
  if (e == cudaSuccess)
    e = dooly::launch_sha256_records(words, rec_off, n, op_bytes, op_off, sym_bytes, sym_off,
                                     attr_digests, out_digest, (cudaStream_t)stream, ctx->n_sm,
                                     &ctx->launches, peers);
  if (e == cudaSuccess)
    e = dooly::launch_peer_sync(peers->n_peers, peers->flag, flag, target, timed_out,
                                (cudaStream_t)stream, &ctx->launches, 0);
  return check_cuda(ctx, e, "sha256_records_bcast");
}

int dooly_enable_peer_access(dooly_ctx* ctx, int peer_device) {
  if (!ctx) return DOOLY_ERR_INVALID_ARG;
  if (peer_device < 0) return fail(ctx, DOOLY_ERR_INVALID_ARG, "enable_peer_access: bad device");
  return check_cuda(ctx, dooly::enable_peer_access(ctx->device, peer_device),
                    "enable_peer_access");
}

int dooly_sha256_messages(dooly_ctx* ctx, const uint8_t* msgs, const int64_t* off, int64_t n,
                          uint8_t* out_digest, void* stream) {
  if (!ctx) return DOOLY_ERR_INVALID_ARG;
  if (n < 0) return fail(ctx, DOOLY_ERR_INVALID_ARG, "sha256_messages: negative size");
  if (n > 0 && (!off || !out_digest))
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "sha256_messages: null pointer");
  DeviceGuard g(ctx->device, __func__);
  if (n > 0) ctx->launches += 1;
  return check_cuda(ctx,
                    dooly::launch_sha256_messages(msgs, off, n, out_digest,
                                                  (cudaStream_t)stream, ctx->n_sm),
                    "sha256_messages");
}

size_t dooly_dedup_workspace_size(int64_t n, int64_t n_db) {
  return dooly::dedup_workspace_size(n, n_db);
}

int dooly_dedup_digests(dooly_ctx* ctx, const uint8_t* digests, int64_t n,
                        const uint8_t* db_digests, int64_t n_db, int64_t* out_first,
                        uint32_t* out_uid, uint8_t* out_is_new, uint8_t* out_in_db,
                        int64_t* out_n_unique, void* workspace, size_t workspace_bytes,
                        void* stream) {
  if (!ctx) return DOOLY_ERR_INVALID_ARG;
  if (n < 0 || n_db < 0) return fail(ctx, DOOLY_ERR_INVALID_ARG, "dedup: negative size");
  if (n + n_db >= (int64_t)0xFFFFFFFF)   // slots hold u32 indices; 0xFFFFFFFF marks empty
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "dedup: more than 2^32-2 digests per call");
  if (!out_n_unique || (n > 0 && (!digests || !out_first || !out_uid || !out_is_new)) ||
      (n_db > 0 && !db_digests))
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "dedup: null pointer");
  if (workspace_bytes < dooly::dedup_workspace_size(n, n_db))
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "dedup: workspace too small");
  DeviceGuard g(ctx->device, __func__);
  return check_cuda(ctx,
                    dooly::launch_dedup(digests, n, db_digests, n_db, out_first, out_uid,
                                        out_is_new, out_in_db, out_n_unique, workspace,
                                        workspace_bytes, (cudaStream_t)stream, ctx->n_sm,
                                        &ctx->launches),
                    "dedup");
}

size_t dooly_route_workspace_size(int64_t n, int world) {
  return dooly::route_workspace_size(n, world);
}

int dooly_route_plan(dooly_ctx* ctx, const uint8_t* digests, int64_t n, int world, int64_t gidx0,
                     int64_t* out_perm, int64_t* out_counts, uint8_t* out_digests,
                     int64_t* out_gidx, void* workspace, size_t workspace_bytes, void* stream) {
  if (!ctx) return DOOLY_ERR_INVALID_ARG;
  if (n < 0 || world < 1 || world > DOOLY_MAX_PEERS + 1 || gidx0 < 0)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "route_plan: bad size or world");
  if (!out_counts || (n > 0 && (!digests || !out_perm || !out_digests || !out_gidx)))
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "route_plan: null pointer");
  if ((uintptr_t)digests % 16 || (uintptr_t)out_digests % 16)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "route_plan: digests must be 16-byte aligned");
  if (!workspace || workspace_bytes < dooly::route_workspace_size(n, world) ||
      (uintptr_t)workspace % 16)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "route_plan: workspace too small or misaligned");
  DeviceGuard g(ctx->device, __func__);
  return check_cuda(ctx,
                    dooly::launch_route_plan(digests, n, world, gidx0, out_perm, out_counts,
                                             out_digests, out_gidx, workspace,
                                             (cudaStream_t)stream, &ctx->launches),
                    "route_plan");
}

int dooly_dedup_firsts(dooly_ctx* ctx, int64_t n, int64_t n_db, const int64_t* gidx,
                       int64_t* out_firsts, void* workspace, size_t workspace_bytes,
                       void* stream) {
  if (!ctx) return DOOLY_ERR_INVALID_ARG;
  if (n < 0 || n_db < 0) return fail(ctx, DOOLY_ERR_INVALID_ARG, "dedup_firsts: negative size");
  if (n > 0 && (!gidx || !out_firsts || !workspace))
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "dedup_firsts: null pointer");
  if (workspace_bytes < dooly::dedup_workspace_size(n, n_db))
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "dedup_firsts: workspace too small");
  DeviceGuard g(ctx->device, __func__);
  return check_cuda(ctx,
                    dooly::launch_dedup_firsts(n, n_db, gidx, out_firsts, workspace,
                                               (cudaStream_t)stream, ctx->n_sm, &ctx->launches),
                    "dedup_firsts");
}

int dooly_route_reply(dooly_ctx* ctx, const int64_t* gidx, const int64_t* first,
                      const uint8_t* is_new, const uint8_t* in_db, int64_t m,
                      const int64_t* all_firsts, int64_t per, int world, int64_t* out_rows,
                      void* stream) {
  if (!ctx) return DOOLY_ERR_INVALID_ARG;
  if (m < 0 || per < 0 || world < 1 || world > DOOLY_MAX_PEERS + 1)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "route_reply: bad size or world");
  if (m > 0 && (!gidx || !first || !is_new || !out_rows || (per > 0 && !all_firsts)))
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "route_reply: null pointer");
  DeviceGuard g(ctx->device, __func__);
  return check_cuda(ctx,
                    dooly::launch_route_reply(gidx, first, is_new, in_db, m, all_firsts, per,
                                              world, out_rows, (cudaStream_t)stream, ctx->n_sm,
                                              &ctx->launches),
                    "route_reply");
}

int dooly_route_finish(dooly_ctx* ctx, const int64_t* rows, const int64_t* perm, int64_t n,
                       int64_t* out_first, uint32_t* out_uid, uint8_t* out_is_new,
                       uint8_t* out_in_db, void* stream) {
  if (!ctx) return DOOLY_ERR_INVALID_ARG;
  if (n < 0) return fail(ctx, DOOLY_ERR_INVALID_ARG, "route_finish: negative size");
  if (n > 0 && (!rows || !perm || !out_first || !out_uid || !out_is_new))
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "route_finish: null pointer");
  DeviceGuard g(ctx->device, __func__);
  return check_cuda(ctx,
                    dooly::launch_route_finish(rows, perm, n, out_first, out_uid, out_is_new,
                                               out_in_db, (cudaStream_t)stream, ctx->n_sm,
                                               &ctx->launches),
                    "route_finish");
}

static int check_oplist(dooly_ctx* ctx, const dooly_oplist* ops, int64_t n_aff, int64_t n_attn,
                        const void* aff_t = nullptr, const void* attn_t = nullptr) {
  if ((uintptr_t)aff_t % 32 != 0 || (uintptr_t)attn_t % 32 != 0)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "regressor tables must be 32-byte aligned");
  if (!ops || ops->n_ops < 0 || ops->n_ops > DOOLY_MAX_OPS)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "oplist: bad n_ops");
  for (int e = 0; e < ops->n_ops; ++e) {
    const int f = ops->feat[e];
    if (f < DOOLY_FEAT_NUM_TOKS || f > DOOLY_FEAT_COMM)
      return fail(ctx, DOOLY_ERR_INVALID_ARG, "oplist: bad feature selector");
    if (f == DOOLY_FEAT_COMM) {
      if (ops->tp < 2) return fail(ctx, DOOLY_ERR_INVALID_ARG, "oplist: comm entry needs tp>=2");
      continue;
    }
    const int64_t lim = f == DOOLY_FEAT_ATTN ? n_attn : n_aff;
    if (ops->row[e] < 0 || ops->row[e] >= lim)
      return fail(ctx, DOOLY_ERR_UNKNOWN_SIGNATURE,
                  "oplist: entry " + std::to_string(e) + " references row " +
                      std::to_string(ops->row[e]) + " outside its regressor table");
  }
  return DOOLY_OK;
}

int dooly_iter_eval(dooly_ctx* ctx, const dooly_oplist* ops, const void* affine_table,
                    int64_t n_affine, const void* attn_table, int64_t n_attn,
                    const uint32_t* it_feat, int64_t n_it, double* it_lat, int64_t* err_first,
                    void* stream) {
  if (!ctx) return DOOLY_ERR_INVALID_ARG;
  int rc = check_oplist(ctx, ops, n_affine, n_attn, affine_table, attn_table);
  if (rc) return rc;
  if (n_it < 0) return fail(ctx, DOOLY_ERR_INVALID_ARG, "iter_eval: negative size");
  if (n_it > 0 && (!it_feat || !it_lat))
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "iter_eval: null pointer");
  DeviceGuard g(ctx->device, __func__);
  if (n_it > 0) ctx->launches += 1;
  return check_cuda(ctx,
                    dooly::launch_iter_eval(ops, affine_table, n_affine, attn_table, n_attn,
                                            it_feat, n_it, it_lat, err_first,
                                            (cudaStream_t)stream, ctx->n_sm),
                    "iter_eval");
}

int dooly_sim_eval(dooly_ctx* ctx, const dooly_oplist* ops, const void* affine_table,
                   int64_t n_affine, const void* attn_table, int64_t n_attn,
                   const uint32_t* it_feat, const double* it_start, const int64_t* it_off,
                   int64_t n_shards, int64_t n_it, const double* arrival,
                   const uint32_t* first_it, const uint32_t* last_it, const uint32_t* out_tok,
                   int64_t n_req, double* it_lat, double* clock, double* ttft, double* tpot,
                   int64_t* err_first, int64_t* req_err_first, void* stream) {
  if (!ctx) return DOOLY_ERR_INVALID_ARG;
  if (n_req < 0 || n_shards < 0)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "sim_eval: negative size");
  if (!it_off) n_shards = n_it > 0 ? 1 : 0;
  if (n_it > 0 && !clock) return fail(ctx, DOOLY_ERR_INVALID_ARG, "sim_eval: null clock");
  if (n_req > 0 && (!arrival || !first_it || !last_it || !out_tok || !ttft || !tpot))
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "sim_eval: null request pointer");
  int rc = dooly_iter_eval(ctx, ops, affine_table, n_affine, attn_table, n_attn, it_feat, n_it,
                           it_lat, err_first, stream);
  if (rc) return rc;
  DeviceGuard g(ctx->device, __func__);
  return check_cuda(ctx,
                    dooly::launch_sim_eval(it_lat, it_start, it_off, n_shards, n_it, clock,
                                           arrival, first_it, last_it, out_tok, n_req, ttft,
                                           tpot, req_err_first, (cudaStream_t)stream, ctx->n_sm,
                                           &ctx->launches),
                    "sim_eval");
}

int dooly_dedup(dooly_ctx* ctx, const uint32_t* words, const int64_t* rec_off, int64_t n,
                const uint8_t* op_bytes, const int64_t* op_off, int64_t n_ops,
                const uint8_t* sym_bytes, const int64_t* sym_off, int64_t n_sym,
                const uint8_t* attr_digests, int64_t n_attr, const uint8_t* db_digests,
                int64_t n_db, uint8_t* out_digest, int64_t* out_first, uint32_t* out_uid,
                uint8_t* out_is_new, uint8_t* out_in_db, int64_t* out_n_unique,
                void* workspace, size_t workspace_bytes, void* stream) {
  if (!ctx) return DOOLY_ERR_INVALID_ARG;
  // Record grouping (dedup.cu): SHA-256 once per distinct packed content, the
  // other records copy their representative's digest.  DOOLY_DEDUP_GROUP=0
  // hashes every record.  Argument errors fall through to the checked calls.
  const char* gv = getenv("DOOLY_DEDUP_GROUP");
  const bool group = (gv == nullptr || gv[0] != '0') && n > 0 && n_db >= 0 &&
                     n + n_db < (int64_t)0xFFFFFFFF && words && rec_off && op_bytes && op_off &&
                     out_digest && workspace &&
                     workspace_bytes >= dooly::dedup_workspace_size(n, n_db);
  int rc;
  if (group) {
    DeviceGuard g(ctx->device, __func__);
    const cudaStream_t st = (cudaStream_t)stream;
    const dooly::RecGroup rg = dooly::rec_group_carve(workspace, n, n_db);
    cudaError_t e = dooly::launch_rec_group(words, rec_off, n, workspace, n_db, st, ctx->n_sm,
                                            &ctx->launches);
    if (e == cudaSuccess)
      e = dooly::launch_sha256_records(words, rec_off, n, op_bytes, op_off, sym_bytes, sym_off,
                                       attr_digests, out_digest, st, ctx->n_sm, &ctx->launches,
                                       nullptr, &rg);
    if (e == cudaSuccess)
      e = dooly::launch_digest_copy(rg.rep, n, out_digest, st, ctx->n_sm, &ctx->launches);
    rc = check_cuda(ctx, e, "dedup: record grouping + sha256");
    if (rc) return rc;
    // records sharing a group share the digest: only the group minima insert
    // (rg.rep = each record's group minimum), the others resolve through it
    if (!out_n_unique || !out_first || !out_uid || !out_is_new || (n_db > 0 && !db_digests))
      return fail(ctx, DOOLY_ERR_INVALID_ARG, "dedup: null pointer");
    return check_cuda(ctx,
                      dooly::launch_dedup(out_digest, n, db_digests, n_db, out_first, out_uid,
                                          out_is_new, out_in_db, out_n_unique, workspace,
                                          workspace_bytes, st, ctx->n_sm, &ctx->launches,
                                          rg.rep),
                      "dedup");
  } else {
    rc = dooly_sha256_records(ctx, words, rec_off, n, op_bytes, op_off, n_ops, sym_bytes,
                              sym_off, n_sym, attr_digests, n_attr, out_digest, stream);
  }
  if (rc) return rc;
  return dooly_dedup_digests(ctx, out_digest, n, db_digests, n_db, out_first, out_uid,
                             out_is_new, out_in_db, out_n_unique, workspace, workspace_bytes,
                             stream);
}

int dooly_profile_fit(dooly_ctx* ctx, int kind, const dooly_sweep_desc* descs, int64_t n_sig,
                      const dooly_sweep_grid* grid, void* table, double* fit_err,
                      uint8_t* status, uint32_t* out_x, double* out_y, const int64_t* out_off,
                      int64_t out_n, void* stream) {
  if (!ctx) return DOOLY_ERR_INVALID_ARG;
  if (kind != DOOLY_KIND_AFFINE && kind != DOOLY_KIND_ATTN)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "profile_fit: unknown kind");
  if (n_sig < 0) return fail(ctx, DOOLY_ERR_INVALID_ARG, "profile_fit: negative size");
  if (!grid || grid->n_tok < 0 || grid->n_tok > DOOLY_SWEEP_MAX || grid->n_req < 0 ||
      grid->n_req > DOOLY_SWEEP_MAX || grid->n_kv < 0 || grid->n_kv > DOOLY_SWEEP_MAX ||
      grid->peak_flops <= 0 || grid->mem_bw <= 0)
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "profile_fit: bad sweep grid");
  if (n_sig > 0 && (!descs || !table || !fit_err || !status))
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "profile_fit: null pointer");
  if ((out_x != nullptr) != (out_y != nullptr) || (out_x != nullptr && out_off == nullptr))
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "profile_fit: out_x/out_y/out_off go together");
  DeviceGuard g(ctx->device, __func__);
  if (n_sig > 0) ctx->launches += 1;
  return check_cuda(ctx,
                    dooly::launch_profile_fit(kind, descs, n_sig, grid, table, fit_err, status,
                                              out_x, out_y, out_off, out_n,
                                              (cudaStream_t)stream, ctx->n_sm),
                    "profile_fit");
}

size_t dooly_sim_workspace_size(const dooly_sched* cfg, int64_t n_req, int64_t n_shards) {
  return dooly::sim_workspace_size(cfg, n_req, n_shards);
}

int dooly_sim_run(dooly_ctx* ctx, const dooly_oplist* ops, const dooly_sched* cfg,
                  const void* affine_table, int64_t n_affine, const void* attn_table,
                  int64_t n_attn, const double* arrival, const uint32_t* prompt,
                  const uint32_t* output, const uint32_t* cached, const int64_t* shard_off,
                  int64_t n_shards, double* ttft, double* tpot, int64_t* n_iter,
                  double* final_clock, int32_t* shard_status, uint32_t* it_log_feat,
                  double* it_log_lat, int64_t it_log_cap, void* workspace,
                  size_t workspace_bytes, void* stream) {
  if (!ctx) return DOOLY_ERR_INVALID_ARG;
  int rc = check_oplist(ctx, ops, n_affine, n_attn, affine_table, attn_table);
  if (rc) return rc;
  if (!cfg || cfg->chunk < 1 || cfg->max_batch < 1 || cfg->max_batch > 1024 ||
      cfg->chunk < cfg->max_batch ||
      cfg->max_iterations < 1 || cfg->kv_capacity_bytes < 0 || cfg->kv_bytes_per_token < 0)
    return fail(ctx, DOOLY_ERR_INVALID_ARG,
                "sim: bad scheduler config (need chunk >= max_batch >= 1)");
  if (n_shards < 0) return fail(ctx, DOOLY_ERR_INVALID_ARG, "sim: negative shard count");
  if (n_shards > 0 && (!shard_off || !n_iter || !final_clock || !shard_status))
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "sim: null pointer");
  if (workspace_bytes < dooly::sim_workspace_size(cfg, 0, n_shards))
    return fail(ctx, DOOLY_ERR_INVALID_ARG, "sim: workspace too small");
  DeviceGuard g(ctx->device, __func__);
  if (n_shards > 0) ctx->launches += 1;
  return check_cuda(
      ctx,
      dooly::launch_sim(ops, cfg, affine_table, n_affine, attn_table, n_attn, arrival, prompt,
                        output, cached, shard_off, n_shards, ttft, tpot, n_iter, final_clock,
                        shard_status, it_log_feat, it_log_lat, it_log_cap, workspace,
                        workspace_bytes, (cudaStream_t)stream, ctx->n_sm),
      "sim_run");
}

}  // extern "C"
