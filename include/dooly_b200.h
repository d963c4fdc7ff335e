/*
 * libdooly_b200 — C-ABI for the B200-native Dooly latency-database hot path.
 *
 * The reference (arxiv/paper_2605_07985, read-only at /root/reference) is pure
 * Python and ships the hot path only as a specification; every entry point
 * below replaces one `[OP]` of that specification, cited as SPEC.md:line.  The
 * Python mirror (paper_2605_07985_b200/{profiler,sim}.py) binds these through
 * ctypes; INTEGRATION.md shows the binding a maintainer adds to pkg/src/dooly.
 *
 * Conventions
 *  - Every pointer argument except `ctx`, `cfg`/`ops` structs and the string
 *    tables noted below is DEVICE memory owned by the caller.
 *  - Calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy default)
 *    and never allocate or synchronise; scratch comes from a caller-provided
 *    workspace sized by the matching *_workspace_size() query.
 *  - Return value: DOOLY_OK or a DOOLY_ERR_* status; message via
 *    dooly_last_error().  Per-item conditions (insufficient data, unknown
 *    signature, extrapolation, clamping) are reported in per-item arrays so
 *    the host wrapper can raise the reference's exception (errors.py:48-85)
 *    after it synchronises.
 *  - A dooly_ctx is bound to one device and is not thread-safe.
 */
#ifndef DOOLY_B200_H
#define DOOLY_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DOOLY_ABI_VERSION 1

/* status codes (mapped to errors.py classes by paper_2605_07985_b200/errors.py) */
#define DOOLY_OK 0
#define DOOLY_ERR_INVALID_ARG 1
#define DOOLY_ERR_INSUFFICIENT_DATA 2  /* errors.py:60 InsufficientData */
#define DOOLY_ERR_UNKNOWN_SIGNATURE 3  /* errors.py:72 UnknownSignature */
#define DOOLY_ERR_DUPLICATE_KEY 4      /* errors.py:52 DuplicateKey */
#define DOOLY_ERR_NON_TERMINATION 5    /* errors.py:84 NonTermination */
#define DOOLY_ERR_CUDA 6
#define DOOLY_ERR_NCCL 7               /* dooly_comm_* (NCCL inside the library) */

/* peer ranks a fused compute + all-gather call can write (8-GPU box) */
#define DOOLY_MAX_PEERS 7

/* regression kinds (App. A.7 of SURVEY.md) */
#define DOOLY_KIND_AFFINE 0 /* [1, f]                      num_toks-type feature  */
#define DOOLY_KIND_ATTN 1   /* [1,f1,f2,f3,f1²,f2²,f3²,f1f2,f1f3,f2f3]  (prefill_toks, batch, kv_tokens) */

/* Regressor tables are arrays of these rows, one per signature (AoS so one
 * predict gathers exactly one 32-B sector / one 128-B line).  A row whose
 * lo[0] > hi[0] is "not fitted" and yields UNKNOWN_SIGNATURE in predict. */
typedef struct {
  double c0, c1;     /* coefficients in the scaled basis f = x * inv_scale   */
  double inv_scale;  /* 1 / max training x (1 if max == 0)                   */
  uint32_t lo, hi;   /* training box (extrapolation flag outside it)         */
} dooly_affine_row;  /* 32 bytes */

typedef struct {
  double c[10];
  double inv_scale[3];
  uint32_t lo[3], hi[3];
} dooly_attn_row; /* 128 bytes */

/* Packed attention table (DOOLY_KIND_ATTN_PACKED): the predict-side form of a
 * dooly_attn_row table, 96 B = 3 sectors per row instead of 4.  The
 * coefficients are stored FOLDED into raw-feature space (inv = 1/hi by IEEE
 * division, 1 if hi == 0) and grouped by feature: sector k = {e_k, a_k, b_k,
 * d_k} holds the terms that multiply feature k first (a: x_k, b: x_k^2,
 * d: x_k x_{k+1 mod 3}), e_0 = c0, e_1 = lo_bits, e_2 = hi_bits
 * (common.cuh fold_row96, oracle/sim.py pack_attn).  Predict evaluates
 *   s_k = ((e'_k + a_k x_k) + b_k x_k^2) + d_k x_k x_{k+1},  p = (s_0 + s_1) + s_2
 * over raw features with no reciprocal; three lanes evaluate one row
 * cooperatively, lane k from sector k.  The box is bit-packed with per-table
 * field widths w[k] (w0+w1+w2 <= 64):
 *   lo_bits = lo0 | lo1 << w0 | lo2 << (w0+w1)   (hi_bits likewise)
 * Unfitted rows: lo_bits = all ones, hi_bits = 0.  Row s lives at
 * packed + 96 * (s + 1); the first 96 B are the header below. */
#define DOOLY_KIND_ATTN_PACKED 2
#define DOOLY_PACK_MAGIC 0x66504144u /* "DAPf": folded coefficients */
typedef struct {
  double w[12]; /* sector k = words 4k..4k+3 = {e_k, a_k, b_k, d_k} */
} dooly_attn_row96; /* 96 bytes */

typedef struct {
  uint32_t magic;      /* DOOLY_PACK_MAGIC once packed                          */
  uint32_t ok;         /* 1 = packable (widths fit, inv == 1/hi on every row)   */
  uint32_t width[3];   /* box field widths, bits                                */
  uint32_t max_hi[3];  /* per-feature max of hi over fitted rows                */
  uint32_t bad_inv;    /* number of fitted rows whose inv_scale != 1/hi         */
  uint32_t pad_;
  int64_t n_sig;
  uint8_t reserved[48];
} dooly_attn_pack_header; /* 96 bytes */

/* per-signature fit status */
#define DOOLY_FIT_OK 0
#define DOOLY_FIT_INSUFFICIENT 1

/* predict flag planes (bit i of word i/32): plane 0 = extrapolated (outside
 * training box), plane 1 = clamped at the 1e-7 s floor */
#define DOOLY_FLAG_PLANES 2

typedef struct dooly_ctx dooly_ctx;

int dooly_version(void);
int dooly_ctx_create(int device, dooly_ctx** out);
void dooly_ctx_destroy(dooly_ctx* ctx);
const char* dooly_last_error(const dooly_ctx* ctx);
/* number of kernels this ctx has launched since creation (host counter) */
int64_t dooly_launch_count(const dooly_ctx* ctx);

/* ------------------------------------------------------------------ K1 dedup
 * Replaces canonicalize, signature_hash
 * and dedup.
 *
 * Packed record (u32 words, little-endian), starting at words[rec_off[i]]:
 *   w0 op_id      index into the op-name table
 *   w1 n_dims | n_sym << 16
 *   w2 attr_id    index into attr-digest table, 0xFFFFFFFF = operator granularity
 *   w3 repeat_count (carried for model_operations rows; not hashed)
 *   n_dims x {pos, val_lo, val_hi}   MODEL_CONFIG dims/scalars, ascending pos
 *   n_sym  x sym_id                  ascending; ids are ranks in bytewise order
 * String tables are device byte arrays with int64 offsets (n+1 entries).
 * The canonical message (sigfmt=1 layout) is rebuilt in registers and hashed;
 * it is never materialised in HBM.
 */
int dooly_sha256_records(dooly_ctx* ctx, const uint32_t* words, const int64_t* rec_off,
                         int64_t n, const uint8_t* op_bytes, const int64_t* op_off,
                         int64_t n_ops, const uint8_t* sym_bytes, const int64_t* sym_off,
                         int64_t n_sym, const uint8_t* attr_digests, int64_t n_attr,
                         uint8_t* out_digest, void* stream);

/* Fused hash + all-gather for the multi-GPU dedup: as
 * dooly_sha256_records, but record i's digest goes to out_digest[row0 + i] (the
 * LOCAL full-size gathered array) and to every peer rank's gathered array at
 * the same row over peer memory; then the arrival counter handshake of
 * dooly_fit_grid_bcast (flag / target / timed_out).  After it every rank holds
 * all ranks' digests in global record order, ready for dooly_dedup_digests. */
typedef struct {
  int32_t n_peers; /* other ranks, 0..DOOLY_MAX_PEERS */
  int32_t pad_;
  int64_t row0;    /* global index of this rank's record 0 */
  uint8_t* digest[DOOLY_MAX_PEERS];
  uint32_t* flag[DOOLY_MAX_PEERS];
} dooly_digest_peers;
int dooly_sha256_records_bcast(dooly_ctx* ctx, const uint32_t* words, const int64_t* rec_off,
                               int64_t n, const uint8_t* op_bytes, const int64_t* op_off,
                               int64_t n_ops, const uint8_t* sym_bytes, const int64_t* sym_off,
                               int64_t n_sym, const uint8_t* attr_digests, int64_t n_attr,
                               uint8_t* out_digest, const dooly_digest_peers* peers,
                               uint32_t* flag, uint32_t target, int32_t* timed_out, void* stream);

/* Let this context's device access `peer_device`'s memory (the fused *_bcast
 * calls store into peer buffers mapped through CUDA IPC): cudaDeviceEnablePeerAccess
 * from the context's device, already-enabled tolerated. */
int dooly_enable_peer_access(dooly_ctx* ctx, int peer_device);

/* Plain SHA-256 of n byte messages (msgs + off[i]..off[i+1]) — signature_hash(bytes). */
int dooly_sha256_messages(dooly_ctx* ctx, const uint8_t* msgs, const int64_t* off, int64_t n,
                          uint8_t* out_digest, void* stream);

/* First-occurrence dedup of n 32-byte digests against an existing DB key set.
 *   out_first[i]  = smallest j with digest[j] == digest[i]
 *   out_uid[i]    = rank of out_first[i] among first occurrences (dense, ordered)
 *   out_is_new[i] = 1 iff i is a first occurrence and its digest is not in db
 *   out_in_db[i]  = 1 iff digest[i] is in db
 *   out_n_unique  = device int64 scalar, number of distinct digests
 * Exact and deterministic for any thread schedule (min-reduction per key). */
size_t dooly_dedup_workspace_size(int64_t n, int64_t n_db);
int dooly_dedup_digests(dooly_ctx* ctx, const uint8_t* digests, int64_t n,
                        const uint8_t* db_digests, int64_t n_db, int64_t* out_first,
                        uint32_t* out_uid, uint8_t* out_is_new, uint8_t* out_in_db,
                        int64_t* out_n_unique, void* workspace, size_t workspace_bytes,
                        void* stream);

/* -------------------------------------------------------------------- K2 fit
 * Replaces fit.  Points of signature s are
 * [pt_off[s], pt_off[s+1]); x is feature-major (kind==ATTN: 3 planes of n_pts
 * u32, AFFINE: 1 plane), y is latency in seconds.  Writes one table row, the
 * training MAPE and a status per signature.  The attention kind uses a
 * moments workspace of dooly_fit_workspace_size(kind, n_sig) bytes (device,
 * 256-B aligned); passing NULL selects the fused single-kernel path. */
size_t dooly_fit_workspace_size(int kind, int64_t n_sig);
int dooly_fit(dooly_ctx* ctx, int kind, const uint32_t* x, int64_t n_pts, const double* y,
              const int64_t* pt_off, int64_t n_sig, void* table, double* fit_err,
              uint8_t* status, void* workspace, size_t workspace_bytes, void* stream);

/* Shared-grid fit: every signature was swept over the SAME n_pts points x
 * (feature-major planes of n_pts u32, the sweep grid of SPEC.md:466-474);
 * y is row-major (n_sig, n_pts) f64.  Same rows, fit_err and statuses as
 * dooly_fit with pt_off[s] = s * n_pts and x repeated per signature, but the
 * Gram matrix, its factor, the scaling and the box are built once.
 * Workspace: dooly_fit_grid_workspace_size(kind, n_pts) bytes of device memory
 * (the shared factor plus the scaled feature planes of the grid). */
size_t dooly_fit_grid_workspace_size(int kind, int64_t n_pts);

/* dooly_fit_grid for attention signatures that also writes the packed 96-byte
 * serving form of the table from the fit epilogue: `packed` receives the
 * dooly_attn_pack_header row followed by one dooly_attn_row96 per signature,
 * byte-identical to dooly_attn_pack(table) (every fitted row carries the
 * shared grid's box, so the field widths are known before the fit).
 * Replaces fit(db) + the serving-table build. */
int dooly_fit_grid_packed(dooly_ctx* ctx, const uint32_t* x, int64_t n_pts, const double* y,
                          int64_t n_sig, void* table, double* fit_err, uint8_t* status,
                          void* packed, void* workspace, size_t workspace_bytes, void* stream);
int dooly_fit_grid(dooly_ctx* ctx, int kind, const uint32_t* x, int64_t n_pts, const double* y,
                   int64_t n_sig, void* table, double* fit_err, uint8_t* status, void* workspace,
                   size_t workspace_bytes, void* stream);

/* Fused fit + all-gather (SURVEY §8(e) "ONE all-gather of the fitted
 * coefficients", done inside the fit instead of as a separate NCCL call).
 * Each rank fits its contiguous signature range [row0, row0 + n_sig) of the
 * global table and its epilogue stores every row, fit_err and status both into
 * the local full-size arrays and into every peer rank's arrays over peer memory
 * (CUDA IPC mappings of the peers' buffers, peer access enabled; NVLink P2P
 * stores on an NVSwitch box).  Then it adds 1 to every rank's arrival counter
 * (flag, system-scope release) and waits, on the stream, until its own
 * counter reaches `target` (= world size x call number): after that the full
 * table is valid on this rank.  The wait gives up after ~20 s and sets
 * *timed_out (device int32) instead of hanging.  table / fit_err / status are
 * the LOCAL full arrays (row0 + s addressing); peers.table[p] etc. the peers'. */
typedef struct {
  int32_t n_peers; /* other ranks, 0..DOOLY_MAX_PEERS */
  int32_t pad_;
  int64_t row0;    /* global row of this rank's signature 0 */
  void* table[DOOLY_MAX_PEERS];
  double* fit_err[DOOLY_MAX_PEERS];
  uint8_t* status[DOOLY_MAX_PEERS];
  uint32_t* flag[DOOLY_MAX_PEERS];
} dooly_grid_peers;
int dooly_fit_grid_bcast(dooly_ctx* ctx, int kind, const uint32_t* x, int64_t n_pts,
                         const double* y, int64_t n_sig, void* table, double* fit_err,
                         uint8_t* status, const dooly_grid_peers* peers, uint32_t* flag,
                         uint32_t target, int32_t* timed_out, void* workspace,
                         size_t workspace_bytes, void* stream);

/* ------------------------------------------------- owner-routed dedup (K1c)
 * The multi-GPU dedup of SURVEY §8(e) with digests routed to their owner
 * rank (owner = last 8 digest bytes as int64 & INT64_MAX, mod world; world <=
 * DOOLY_MAX_PEERS + 1), every step a device kernel:
 *   dooly_route_plan   stable counting sort of n local digests by owner:
 *                      out_perm[j] = local index of routed row j, out_counts
 *                      [world] rows per owner, out_digests / out_gidx the rows
 *                      (global index gidx0 + i) in bucket order — the send
 *                      buffers of the all-to-all (dooly_alltoallv);
 *   (owner)            dooly_dedup_digests on the received digests (+ its
 *                      share of the DB keys, planned the same way), then
 *   dooly_dedup_firsts its first occurrences' global indices in order
 *                      (same workspace, right after the dedup);
 *   dooly_route_reply  per received row (global first, global uid, is_new |
 *                      in_db << 1) as 3 int64; uid = number of first
 *                      occurrences over all owners with a smaller global index
 *                      (all_firsts: world sorted lists of `per` entries padded
 *                      with INT64_MAX, the all-gather of every owner's firsts);
 *   dooly_route_finish the replies (all-to-all back, bucket order) scattered
 *                      through out_perm into first / uid / is_new / in_db.
 * Equal to dooly_dedup_digests over the whole global list, bit for bit. */
size_t dooly_route_workspace_size(int64_t n, int world);
int dooly_route_plan(dooly_ctx* ctx, const uint8_t* digests, int64_t n, int world, int64_t gidx0,
                     int64_t* out_perm, int64_t* out_counts, uint8_t* out_digests,
                     int64_t* out_gidx, void* workspace, size_t workspace_bytes, void* stream);
int dooly_dedup_firsts(dooly_ctx* ctx, int64_t n, int64_t n_db, const int64_t* gidx,
                       int64_t* out_firsts, void* workspace, size_t workspace_bytes,
                       void* stream);
int dooly_route_reply(dooly_ctx* ctx, const int64_t* gidx, const int64_t* first,
                      const uint8_t* is_new, const uint8_t* in_db, int64_t m,
                      const int64_t* all_firsts, int64_t per, int world, int64_t* out_rows,
                      void* stream);
int dooly_route_finish(dooly_ctx* ctx, const int64_t* rows, const int64_t* perm, int64_t n,
                       int64_t* out_first, uint32_t* out_uid, uint8_t* out_is_new,
                       uint8_t* out_in_db, void* stream);

/* ------------------------------------------------------------ communicator
 * NCCL inside the library: the NCCL forms of the multi-GPU
 * exchanges beside the fused peer-memory ones.  Replaces the reference's
 * nothing — the reference is single-process Python; these are the
 * exports §8(b) names.  Failures return DOOLY_ERR_NCCL, message via
 * dooly_comm_last_error (NULL comm: the calling thread's last failure).
 *   one process per GPU: rank 0 gets the id (dooly_comm_unique_id), the caller
 *     ships the DOOLY_COMM_ID_BYTES to every rank, each rank calls
 *     dooly_comm_init_rank(device, id, nranks, rank);
 *   one process, ndev GPUs: dooly_comm_create (ncclCommInitAll).
 * dooly_allgather is in place: bufs[i] (local device i) holds nranks blocks of
 * bytes_per_rank, its own at (rank0 + i) x bytes_per_rank.  dooly_alltoallv
 * (one local device) sends block p of `send` to rank p and receives block p of
 * `recv` from it; counts are HOST arrays of nranks element counts. */
#define DOOLY_COMM_ID_BYTES 128
typedef struct dooly_comm dooly_comm;
int dooly_comm_unique_id(uint8_t* out_id);
int dooly_comm_init_rank(int device, const uint8_t* id, int nranks, int rank, dooly_comm** out);
int dooly_comm_create(int ndev, const int* devs, dooly_comm** out);
void dooly_comm_destroy(dooly_comm* comm);
const char* dooly_comm_last_error(const dooly_comm* comm);
int dooly_comm_size(const dooly_comm* comm, int* nranks, int* rank0, int* n_local);
int dooly_allgather(dooly_comm* comm, void* const* bufs, size_t bytes_per_rank,
                    void* const* streams);
int dooly_alltoallv(dooly_comm* comm, const void* send, const int64_t* send_counts, void* recv,
                    const int64_t* recv_counts, size_t elem_bytes, void* stream);

/* ---------------------------------------------------------------- K3 predict
 * Replaces predict.  sig[i] indexes the table; x is
 * feature-major (planes of n_q u32).  out[i] = max(poly, 1e-7) evaluated
 * mul-then-add without contraction; flag_bits holds DOOLY_FLAG_PLANES planes
 * of ceil(n_q/32) words (may be NULL).  Queries on unknown/unfitted rows write
 * NaN and atomically min their index into *err_first (device int64, caller
 * initialises to INT64_MAX; may be NULL). */
int dooly_predict(dooly_ctx* ctx, int kind, const void* table, int64_t n_sig,
                  const uint32_t* sig, const uint32_t* x, int64_t n_q, double* out,
                  uint32_t* flag_bits, int64_t* err_first, void* stream);

/* Convert an attention table (n_sig dooly_attn_row) into the packed predict
 * form (DOOLY_KIND_ATTN_PACKED) at `packed` (dooly_attn_pack_bytes(n_sig)
 * bytes, 32-B aligned).  Asynchronous; the caller reads header.ok after the
 * stream syncs.  dooly_predict on a header with ok != 1 flags every query as
 * unknown (NaN + err_first), never silently mispredicts. */
size_t dooly_attn_pack_bytes(int64_t n_sig);
int dooly_attn_pack(dooly_ctx* ctx, const void* table, int64_t n_sig, void* packed,
                    void* stream);

/* ------------------------------------------------------- K5 fused sweep -> fit
 * evaluates the analytical latency model (SPEC.md:476-484,
 * op formulas of profiler.op_cost) over each signature's sweep grid
 * (App. A.5) in registers and fits it (K2 semantics) without
 * materialising measurements.  descs is DEVICE memory (n_sig entries), grid
 * is a HOST struct passed by value.  out_x/out_y/out_off (device, optional)
 * receive the generated points (feature-major planes of out_n) for checking. */
#define DOOLY_OP_RESHAPE 0
#define DOOLY_OP_LINEAR 1     /* dim: K, N                        */
#define DOOLY_OP_EMBEDDING 2  /* dim: hidden                      */
#define DOOLY_OP_RMSNORM 3    /* dim: hidden                      */
#define DOOLY_OP_ROTARY 4     /* dim: hq*d + hkv*d                */
#define DOOLY_OP_ACT_MUL 5    /* dim: 2*intermediate              */
#define DOOLY_OP_TOPK 6       /* dim: experts                     */
#define DOOLY_OP_MOE 7        /* dim: experts, 2*expert_inter, hidden, top_k */
#define DOOLY_OP_ATTENTION 8  /* dim: hq, head_dim, hkv           */
#define DOOLY_SWEEP_MAX 16
typedef struct {
  int32_t op;           /* DOOLY_OP_*                                         */
  int32_t feature;      /* DOOLY_FEAT_NUM_TOKS / NUM_SEQS / ATTN               */
  int64_t dim[4];
  int32_t window;       /* attention sliding window, 0 = full                  */
  int32_t dtype_bytes;
  int64_t max_context;
  double mult[2];       /* cost multiplier: [prefill or all, decode]           */
} dooly_sweep_desc;
typedef struct {
  int32_t n_tok, n_req, n_kv, pad_;
  int64_t chunk, max_batch;
  uint32_t tok[DOOLY_SWEEP_MAX], req[DOOLY_SWEEP_MAX], kv[DOOLY_SWEEP_MAX];
  double peak_flops, mem_bw, overhead;
} dooly_sweep_grid;
int dooly_profile_fit(dooly_ctx* ctx, int kind, const dooly_sweep_desc* descs, int64_t n_sig,
                      const dooly_sweep_grid* grid, void* table, double* fit_err,
                      uint8_t* status, uint32_t* out_x, double* out_y, const int64_t* out_off,
                      int64_t out_n, void* stream);

/* ------------------------------------------------------------------- K4 sim
 * Call-graph op list for one (model, backend, tp): iter_latency
 *   lat = sum_e repeat_e * max(pred_e(x_it), 1e-7)   [in list order]
 *       + sum_c repeat_c * comm(tp, num_toks * bytes_per_tok_c)
 * HOST struct; the arrays it points to are HOST memory (copied to device
 * constant memory at launch). */
#define DOOLY_MAX_OPS 64
#define DOOLY_FEAT_NUM_TOKS 0    /* affine on tokens scheduled this iteration     */
#define DOOLY_FEAT_NUM_SEQS 1    /* affine on requests in the iteration (lm_head) */
#define DOOLY_FEAT_ATTN 2        /* attention (prefill_toks, batch, kv_tokens[w]) */
#define DOOLY_FEAT_COMM 3        /* ring all-reduce of num_toks*bytes_per_tok     */
typedef struct {
  int32_t n_ops;
  int32_t tp;
  double comm_alpha, comm_beta;
  int32_t feat[DOOLY_MAX_OPS];      /* DOOLY_FEAT_*                                */
  int32_t row[DOOLY_MAX_OPS];       /* table row (affine table or attention table) */
  int32_t repeat[DOOLY_MAX_OPS];
  int32_t window_slot[DOOLY_MAX_OPS]; /* ATTN: 0 = full kv, 1 = windowed kv       */
  int64_t bytes_per_tok[DOOLY_MAX_OPS]; /* COMM                                   */
} dooly_oplist;

/* Per-iteration features, 5 planes of n_it u32 (feature-major):
 *   0 num_toks, 1 prefill_toks, 2 batch, 3 kv_tokens (full), 4 kv_tokens (windowed) */
#define DOOLY_IT_FEATS 5
int dooly_iter_eval(dooly_ctx* ctx, const dooly_oplist* ops, const void* affine_table,
                    int64_t n_affine, const void* attn_table, int64_t n_attn,
                    const uint32_t* it_feat, int64_t n_it, double* it_lat,
                    int64_t* err_first, void* stream);

/* Device-resident serving loop: one CTA per
 * independent replica shard runs FCFS continuous batching with chunked
 * prefill, the fused gather-evaluate-reduce iteration latency above, the f64
 * clock, and stamps per-request first/last-token times. */
typedef struct {
  int32_t chunk;            /* prefill token budget per iteration (decodes count, D1) */
  int32_t max_batch;
  int32_t window;           /* sliding window of the windowed kv plane (0 = none)     */
  int32_t pad_;
  int64_t kv_bytes_per_token;
  int64_t kv_capacity_bytes; /* admission cap on reserved (prompt+output) KV bytes    */
  int64_t max_iterations;   /* per shard NonTermination guard                         */
} dooly_sched;

/* Requests of shard s are [shard_off[s], shard_off[s+1]), sorted by arrival.
 * Outputs per request (device f64): ttft = first-token time - arrival, tpot =
 * (last - first token time) / (output - 1) (NaN when output < 2).  Per shard:
 * iteration count, final clock, status (DOOLY_OK, DOOLY_ERR_NON_TERMINATION
 * when max_iterations is hit, DOOLY_ERR_INVALID_ARG when the head request can
 * never fit the KV capacity, DOOLY_ERR_UNKNOWN_SIGNATURE for unfitted rows).
 * Optional it_log (device, may be NULL): per shard up to it_log_cap rows of
 * DOOLY_IT_FEATS u32 features + the f64 iteration latency, for verification.
 * The workspace is currently unused (all scheduler state lives in shared
 * memory; max_batch <= 1024). */
size_t dooly_sim_workspace_size(const dooly_sched* cfg, int64_t n_req, int64_t n_shards);
int dooly_sim_run(dooly_ctx* ctx, const dooly_oplist* ops, const dooly_sched* cfg,
                  const void* affine_table, int64_t n_affine, const void* attn_table,
                  int64_t n_attn, const double* arrival, const uint32_t* prompt,
                  const uint32_t* output, const uint32_t* cached, const int64_t* shard_off,
                  int64_t n_shards, double* ttft, double* tpot, int64_t* n_iter,
                  double* final_clock, int32_t* shard_status, uint32_t* it_log_feat,
                  double* it_log_lat, int64_t it_log_cap, void* workspace,
                  size_t workspace_bytes, void* stream);

/* Host-scheduled evaluation (SURVEY §8(b) dooly_sim_eval): an external
 * scheduler supplies the iterations; the device evaluates them and derives the
 * request metrics.
 *   it_feat   DOOLY_IT_FEATS planes of n_it u32 (as dooly_iter_eval)
 *   it_start  per iteration, the earliest start (the arrival an idle replica
 *             jumps to), 0 when the replica was busy; NULL = 0
 *   it_off    n_shards + 1 offsets of independent replica shards (NULL: one)
 *   clock[i]  = max(clock[i-1], it_start[i]) + it_lat[i], sequential f64 per
 *               shard, bit-identical to the event loop's clock
 *   first_it / last_it  global iteration that produced a request's first /
 *             last token (0xFFFFFFFF = never)
 *   ttft      = clock[first_it] - arrival;  tpot = (clock[last_it] -
 *               clock[first_it]) / (out_tok - 1), NaN when out_tok < 2
 * err_first  (optional) first iteration on an unknown regressor row
 * req_err_first (optional) first request with an out-of-range iteration index
 * it_lat and clock are caller-owned device outputs of n_it f64. */
int dooly_sim_eval(dooly_ctx* ctx, const dooly_oplist* ops, const void* affine_table,
                   int64_t n_affine, const void* attn_table, int64_t n_attn,
                   const uint32_t* it_feat, const double* it_start, const int64_t* it_off,
                   int64_t n_shards, int64_t n_it, const double* arrival,
                   const uint32_t* first_it, const uint32_t* last_it, const uint32_t* out_tok,
                   int64_t n_req, double* it_lat, double* clock, double* ttft, double* tpot,
                   int64_t* err_first, int64_t* req_err_first, void* stream);

/* canonicalize + signature_hash + dedup in one call (SURVEY §8(b) dooly_dedup):
 * dooly_sha256_records into out_digest, then dooly_dedup_digests.  The
 * workspace is dooly_dedup_workspace_size(n, n_db) bytes. */
int dooly_dedup(dooly_ctx* ctx, const uint32_t* words, const int64_t* rec_off, int64_t n,
                const uint8_t* op_bytes, const int64_t* op_off, int64_t n_ops,
                const uint8_t* sym_bytes, const int64_t* sym_off, int64_t n_sym,
                const uint8_t* attr_digests, int64_t n_attr, const uint8_t* db_digests,
                int64_t n_db, uint8_t* out_digest, int64_t* out_first, uint32_t* out_uid,
                uint8_t* out_is_new, uint8_t* out_in_db, int64_t* out_n_unique,
                void* workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DOOLY_B200_H */
