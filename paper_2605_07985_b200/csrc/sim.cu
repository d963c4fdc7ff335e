// K4 — fused gather-evaluate-reduce iteration latency (iter_latency,
// SPEC.md:586-594) and the device-resident serving loop (run, SPEC.md:596-604;
// schedule_step).
//
// iter_eval: one thread per iteration; the op list's regressor rows are staged
//   once per CTA in shared memory, so each iteration is a pure in-SM
//   gather/evaluate/reduce over the call graph.
//
// sim_run: one WARP per independent replica shard (App. A.14).  Each shard's
//   event loop is inherently sequential (the clock decides admissions), so the
//   parallelism is across shards, and inside a shard across the running batch
//   (lanes own running slots) and across op-list entries (lanes own entries).
//   The scheduler state lives in shared memory; the per-iteration loop touches
//   HBM only to read newly admitted requests and to write TTFT/TPOT.  One loop
//   pass per admission: the scheduled iteration is window iteration 0, and
//   when the rest of the window's composition is fixed (everything decoding,
//   no admission possible before an arrival or a finish) lanes 1..31 evaluate
//   the following iterations in parallel, finishes included; the clock then
//   commits them in order (profiles/r2_sim_window.md).
//
// Parity: per-entry predictions use the same no-FMA evaluation as predict
//   (common.cuh); the per-iteration sum runs in op-list order on lane 0 with
//   separate mul/add, and the clock is a sequential f64 accumulation — the
//   exact arithmetic sequence of oracle/sim.py, so iteration latencies, the
//   clock, every admission decision and therefore TTFT/TPOT match bit-for-bit
//   given the same regressor rows.
//
// Scheduler invariant used (proved in DESIGN.md "sim"): at the start of an
// iteration the running list is [decode-phase ... | at most one prefill-phase
// request], because prefill budget is granted in running order and admission
// stops as soon as the budget is exhausted.
#include <cstdlib>

#include "common.cuh"

namespace dooly {

#ifndef SIM_WARPS_N
#define SIM_WARPS_N 4  // replicas (warps) per CTA
#endif
constexpr int SIM_WARPS = SIM_WARPS_N;
#ifndef SIM_UNROLL
#define SIM_UNROLL 2  // unroll of the per-slot passes (2: C4 60.9 -> 58.7 ms; 4: 59.5)
#endif
constexpr int kSimUnroll = SIM_UNROLL;

// The op list staged in shared memory: regressor rows, and the per-entry
// fields (feature, repeat, window slot, comm bytes per token) so that lanes
// evaluating DIFFERENT entries read shared memory instead of issuing
// lane-divergent loads from the kernel-parameter bank (which serialise per
// distinct address); the comm constants 2(tp-1)/tp and 1/tp are formed once.
struct StagedOps {
  AffineRow aff[DOOLY_MAX_OPS];
  AttnRow attn[DOOLY_MAX_OPS];
  int32_t feat[DOOLY_MAX_OPS];
  int32_t wslot[DOOLY_MAX_OPS];
  double rep[DOOLY_MAX_OPS];
  uint64_t bpt[DOOLY_MAX_OPS];
  double comm_a;    // RN(2(tp-1) / tp)
  double comm_rtp;  // RN(1 / tp) when tp is a power of two (exact scaling), else 0
  // entries grouped by kind (op-list order within a kind) for the window's
  // straight-line evaluation: [0, n_aff) affine, then attention, then comm
  uint8_t kidx[DOOLY_MAX_OPS];
  int n_aff, n_att;
};

__device__ __forceinline__ void stage_ops(const dooly_oplist& ops, const void* aff_t,
                                          const void* attn_t, StagedOps* s, int tid, int nthr) {
  for (int e = tid; e < ops.n_ops; e += nthr) {
    const int f = ops.feat[e];
    s->feat[e] = f;
    s->wslot[e] = ops.window_slot[e];
    s->rep[e] = (double)ops.repeat[e];
    s->bpt[e] = (uint64_t)ops.bytes_per_tok[e];
    if (f == DOOLY_FEAT_ATTN)
      s->attn[e] = load_attn(static_cast<const dooly_attn_row*>(attn_t), ops.row[e]);
    else if (f != DOOLY_FEAT_COMM)
      s->aff[e] = load_affine(static_cast<const dooly_affine_row*>(aff_t), ops.row[e]);
  }
  if (tid == 0) {
    int k = 0;
    for (int pass = 0; pass < 3; ++pass) {
      for (int e = 0; e < ops.n_ops; ++e) {
        const int f = ops.feat[e];
        const int cls = f == DOOLY_FEAT_ATTN ? 1 : f == DOOLY_FEAT_COMM ? 2 : 0;
        if (cls == pass) s->kidx[k++] = (uint8_t)e;
      }
      if (pass == 0) s->n_aff = k;
      if (pass == 1) s->n_att = k - s->n_aff;
    }
    const int tp = ops.tp > 0 ? ops.tp : 1;
    s->comm_a = __ddiv_rn((double)(2 * (tp - 1)), (double)tp);
    s->comm_rtp = (tp & (tp - 1)) == 0 ? __drcp_rn((double)tp) : 0.0;
  }
}

// comm_latency: 2(tp-1)/tp * (alpha + bytes/tp * beta), evaluated
// in Python's operator order (a = RN(2(tp-1)/tp) and, for a power-of-two tp,
// bytes/tp as the exact scaling by RN(1/tp) — both staged once).
__device__ __forceinline__ double comm_latency(const StagedOps* s, int tp, double alpha,
                                               double beta, uint64_t bytes) {
  const double q = s->comm_rtp != 0.0 ? mul((double)bytes, s->comm_rtp)
                                      : __ddiv_rn((double)bytes, (double)tp);
  const double b = mul(q, beta);
  return mul(s->comm_a, add(alpha, b));
}

// One entry's clamped contribution before the repeat multiply; invalid rows -> NaN.
__device__ __forceinline__ double entry_value(const dooly_oplist& ops, const StagedOps* s, int e,
                                              uint32_t num_toks, uint32_t prefill, uint32_t batch,
                                              uint32_t kv_full, uint32_t kv_win, bool& bad) {
  const int f = s->feat[e];
  bool cl;
  if (f == DOOLY_FEAT_COMM)
    return comm_latency(s, ops.tp, ops.comm_alpha, ops.comm_beta, (uint64_t)num_toks * s->bpt[e]);
  if (f == DOOLY_FEAT_ATTN) {
    const AttnRow& r = s->attn[e];
    if (!attn_valid(r)) {
      bad = true;
      return nan64();
    }
    return clamp_floor(eval_attn(r, prefill, batch, s->wslot[e] ? kv_win : kv_full), cl);
  }
  const AffineRow& r = s->aff[e];
  if (!affine_valid(r)) {
    bad = true;
    return nan64();
  }
  return clamp_floor(eval_affine(r, f == DOOLY_FEAT_NUM_SEQS ? batch : num_toks), cl);
}

__global__ void __launch_bounds__(256) iter_eval_kernel(
    const dooly_oplist ops, const void* __restrict__ aff_t, const void* __restrict__ attn_t,
    const uint32_t* __restrict__ feat, int64_t n_it, double* __restrict__ out,
    int64_t* __restrict__ err_first) {
  __shared__ StagedOps s;
  stage_ops(ops, aff_t, attn_t, &s, threadIdx.x, blockDim.x);
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_it; i += stride) {
    const uint32_t nt = feat[i], pf = feat[n_it + i], bt = feat[2 * n_it + i],
                   kv = feat[3 * n_it + i], kw = feat[4 * n_it + i];
    double lat = 0.0;
    bool bad = false;
    for (int e = 0; e < ops.n_ops; ++e) {
      const double v = entry_value(ops, &s, e, nt, pf, bt, kv, kw, bad);
      lat = add(lat, mul(s.rep[e], v));
    }
    out[i] = lat;
    if (bad && err_first) atomicMin(reinterpret_cast<unsigned long long*>(err_first), (unsigned long long)i);
  }
}

cudaError_t launch_iter_eval(const dooly_oplist* ops, const void* aff, int64_t n_aff,
                             const void* attn, int64_t n_attn, const uint32_t* it_feat,
                             int64_t n_it, double* it_lat, int64_t* err_first,
                             cudaStream_t stream, int n_sm) {
  (void)n_aff;
  (void)n_attn;
  if (n_it == 0) return cudaSuccess;
  int64_t blocks = (n_it + 255) / 256;
  if (blocks > (int64_t)n_sm * 8) blocks = (int64_t)n_sm * 8;
  iter_eval_kernel<<<(unsigned)blocks, 256, 0, stream>>>(*ops, aff, attn, it_feat, n_it, it_lat,
                                                         err_first);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ sim_run

struct SlotArrays {  // per-warp views into dynamic shared memory
  uint32_t* rq;      // request index within the shard
  uint32_t* left;    // prefill tokens still to schedule
  uint32_t* dec;     // output tokens produced
  uint32_t* kv;      // tokens in the KV cache before this iteration
  uint32_t* out;     // output length (copied at admission: no HBM read per iteration)
  uint32_t* ptot;    // prompt + output tokens (its KV reservation / kv_bytes_per_token)
  double* t_first;   // first-token time
  double* arr;       // arrival time
  uint32_t* wb;      // window scratch: KV tokens at window iteration u >= 1 are wb + u
  uint32_t* wr;      // window scratch: iterations the slot runs from the window's start
};
constexpr int kSlotBytes = 48;  // 2 x f64 + 8 x u32 per running slot

size_t sim_workspace_size(const dooly_sched* cfg, int64_t n_req, int64_t n_shards) {
  (void)cfg;
  (void)n_req;
  (void)n_shards;
  return 0;  // all scheduler state is in shared memory
}

__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t v) {
  return __reduce_add_sync(0xFFFFFFFFu, v);
}

// One iteration's latency by a single lane, entries evaluated grouped by kind
// with no data-dependent branch inside a group (4 affine or 2 attention
// entries per straight-line step, so their FP64 chains overlap), each repeat
// product parked in the lane's column of pv (entry-major, 32 doubles per
// entry), then the sum in op-list order.  Every entry value and product is
// the same IEEE operation sequence as entry_value / the serial path.
__device__ __forceinline__ double window_latency(const dooly_oplist& ops, const StagedOps* s,
                                                 double* pv, int lane, uint32_t nt, uint32_t pf,
                                                 uint32_t bt, uint32_t ks, uint32_t kw,
                                                 bool& bad) {
  const int na = s->n_aff, nat = s->n_att, n = ops.n_ops;
  for (int i = 0; i < na; i += 4) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = s->kidx[min(i + k, na - 1)];  // the tail repeats the last entry
      const AffineRow& r = s->aff[e];
      bad |= !affine_valid(r);
      bool cl;
      const double v = clamp_floor(eval_affine(r, s->feat[e] == DOOLY_FEAT_NUM_SEQS ? bt : nt), cl);
      pv[e * 32 + lane] = mul(s->rep[e], v);
    }
  }
  for (int i = 0; i < nat; i += 2) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int e = s->kidx[na + min(i + k, nat - 1)];
      const AttnRow& r = s->attn[e];
      bad |= !attn_valid(r);
      bool cl;
      const double v = clamp_floor(eval_attn(r, pf, bt, s->wslot[e] ? kw : ks), cl);
      pv[e * 32 + lane] = mul(s->rep[e], v);
    }
  }
  for (int i = na + nat; i < n; ++i) {
    const int e = s->kidx[i];
    pv[e * 32 + lane] =
        mul(s->rep[e], comm_latency(s, ops.tp, ops.comm_alpha, ops.comm_beta, (uint64_t)nt * s->bpt[e]));
  }
  double lat = 0.0;
#pragma unroll 4
  for (int e = 0; e < n; ++e) lat = add(lat, pv[e * 32 + lane]);
  return lat;
}

__global__ void __launch_bounds__(SIM_WARPS * 32) sim_run_kernel(
    const dooly_oplist ops, const dooly_sched cfg, const void* __restrict__ aff_t,
    const void* __restrict__ attn_t, const double* __restrict__ arrival,
    const uint32_t* __restrict__ prompt, const uint32_t* __restrict__ output,
    const uint32_t* __restrict__ cached, const int64_t* __restrict__ shard_off, int64_t n_shards,
    double* __restrict__ ttft, double* __restrict__ tpot, int64_t* __restrict__ n_iter_out,
    double* __restrict__ clock_out, int32_t* __restrict__ status_out,
    uint32_t* __restrict__ log_feat, double* __restrict__ log_lat, int64_t log_cap, int use_pv) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ StagedOps s_ops;
  __shared__ __align__(16) double s_sum[SIM_WARPS][64];  // per-entry products / window latencies
  __shared__ uint32_t s_hc[SIM_WARPS][32], s_hk[SIM_WARPS][32];  // window finish histograms
  stage_ops(ops, aff_t, attn_t, &s_ops, threadIdx.x, blockDim.x);
  __syncthreads();

  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int MB = cfg.max_batch;
  SlotArrays sl;
  {
    unsigned char* p = dyn + (size_t)wid * MB * kSlotBytes;
    sl.t_first = reinterpret_cast<double*>(p);
    sl.arr = sl.t_first + MB;
    sl.rq = reinterpret_cast<uint32_t*>(p + (size_t)MB * 16);
    sl.left = sl.rq + MB;
    sl.dec = sl.left + MB;
    sl.kv = sl.dec + MB;
    sl.out = sl.kv + MB;
    sl.ptot = sl.out + MB;
    sl.wb = sl.ptot + MB;
    sl.wr = sl.wb + MB;
  }
  // after the slot arrays, if launched with room (use_pv):
  //  2: the decode-product table P[x][e] = repeat_e x value_e(num_toks = batch = x) of every
  //     affine and comm entry for x in [0, MB], shared by the CTA's warps — a window
  //     iteration u >= 1 is pure decode with num_toks = batch = nr(u) <= MB, so its
  //     non-attention products are table reads (the same IEEE operations, done once);
  //  1: per-lane product columns for window_latency.
  double* pv_base = use_pv == 1 ? reinterpret_cast<double*>(dyn + (size_t)SIM_WARPS * MB * kSlotBytes)
                                : nullptr;
  double* ptab = use_pv == 2 ? reinterpret_cast<double*>(dyn + (size_t)SIM_WARPS * MB * kSlotBytes)
                             : nullptr;
  if (ptab != nullptr) {
    const int no = ops.n_ops;
    for (int idx = threadIdx.x; idx < (MB + 1) * no; idx += blockDim.x) {
      const int e = idx % no;
      const uint32_t x = (uint32_t)(idx / no);
      const int f = s_ops.feat[e];
      double v = 0.0;
      if (f == DOOLY_FEAT_COMM) {
        v = mul(s_ops.rep[e], comm_latency(&s_ops, ops.tp, ops.comm_alpha, ops.comm_beta,
                                           (uint64_t)x * s_ops.bpt[e]));
      } else if (f != DOOLY_FEAT_ATTN) {
        bool cl;
        v = mul(s_ops.rep[e], clamp_floor(eval_affine(s_ops.aff[e], x), cl));
      }
      ptab[idx] = v;
    }
    __syncthreads();
  }
  const uint32_t W = cfg.window > 0 ? (uint32_t)cfg.window : 0u;
  const uint64_t kvb = (uint64_t)cfg.kv_bytes_per_token;
  const uint64_t cap = (uint64_t)cfg.kv_capacity_bytes;

  for (int64_t shard = (int64_t)blockIdx.x * SIM_WARPS + wid; shard < n_shards;
       shard += (int64_t)gridDim.x * SIM_WARPS) {
    const int64_t base = shard_off[shard];
    const int64_t n = shard_off[shard + 1] - base;
    const double* arr = arrival + base;
    const uint32_t* pr = prompt + base;
    const uint32_t* ou = output + base;
    const uint32_t* ca = cached + base;
    double clock = 0.0;
    int64_t arrive = 0, admit = 0, it = 0;
    int nrun = 0;
    uint64_t reserved = 0;
    int32_t status = DOOLY_OK;
    // Prefetch windows (registers, lane = offset): the arrival times from
    // `arrive` on, and the waiting requests' (prompt, output, cached, arrival)
    // from `wbase` on.  They are reloaded right after they are consumed and
    // first read in the NEXT iteration, so the HBM/L2 latency overlaps an
    // iteration's work instead of sitting on the critical path.
    auto ld_arr = [&](int64_t i0) { return i0 + lane < n ? arr[i0 + lane] : 0.0; };
    double win_arr = ld_arr(0);
    int64_t wbase = 0;
    uint32_t w_p = 0, w_o = 0, w_c = 0;
    double w_a = 0.0;
    auto ld_wait = [&](int64_t i0) {
      wbase = i0;
      const int64_t i = i0 + lane;
      if (i < n) {
        w_p = pr[i];
        w_o = ou[i];
        w_c = ca[i];
        w_a = arr[i];
      }
    };
    ld_wait(0);

#ifdef SIM_PASS_COUNT
    int64_t passes = 0;  // diagnostic build: loop passes instead of iterations in n_iter_out
#endif
    while (true) {
#ifdef SIM_PASS_COUNT
      ++passes;
#endif
      // ---- 1. arrivals with arrival <= clock (sorted: a ballot prefix)
      double next_arr = __shfl_sync(0xFFFFFFFFu, win_arr, 0);
      if (arrive < n && next_arr <= clock) {
        while (true) {
          const bool in = arrive + lane < n && win_arr <= clock;
          const uint32_t b = __ballot_sync(0xFFFFFFFFu, in);
          const int cnt = __popc(b);  // prefix because arrivals are sorted
          arrive += cnt;
          win_arr = ld_arr(arrive);
          if (cnt < 32) break;
        }
      }
      if (nrun == 0 && admit == arrive) {
        if (arrive == n) break;
        clock = __shfl_sync(0xFFFFFFFFu, win_arr, 0);  // idle: jump to the next arrival (exact copy)
        continue;
      }
      if (it >= cfg.max_iterations) {  // work remains but the cap is reached
        status = DOOLY_ERR_NON_TERMINATION;
        break;
      }
      // ---- 2. schedule (decode prefix | <=1 prefill at the tail)
      const bool has_p = nrun > 0 && sl.left[nrun - 1] > 0;
      const int n_dec = nrun - (has_p ? 1 : 0);
      int64_t budget = (int64_t)cfg.chunk - n_dec;
      uint32_t take_p = 0;
      if (has_p) {
        const uint32_t l = sl.left[nrun - 1];
        take_p = (int64_t)l < budget ? l : (uint32_t)budget;
        budget -= take_p;
      }
      // admissions: lanes prefetch the next 32 waiting requests, lane 0 decides serially
      const int nrun0 = nrun;
      uint32_t adm_pf = 0, adm_tok = 0, adm_kv = 0, adm_kvw = 0;
      int n_adm = 0;
      bool blocked = false;       // the FCFS head does not fit the KV capacity
      bool adm_partial = false;   // an admitted prompt keeps prefilling after this iteration
      while (admit < arrive && nrun < MB && budget > 0) {
        if (wbase != admit) ld_wait(admit);  // only after 32 admissions in one iteration
        int took = 0;  // admitted in this round (uniform after broadcast)
        for (int k = 0; k < 32; ++k) {
          if (admit + k >= arrive || nrun + took >= MB || budget <= 0) break;
          const uint32_t p = __shfl_sync(0xFFFFFFFFu, w_p, k);
          const uint32_t o = __shfl_sync(0xFFFFFFFFu, w_o, k);
          const uint32_t c = __shfl_sync(0xFFFFFFFFu, w_c, k);
          const double a = __shfl_sync(0xFFFFFFFFu, w_a, k);
          const uint64_t need = (uint64_t)(p + o) * kvb;
          if (reserved + need > cap) {
            blocked = true;
            break;
          }
          const uint32_t work = p - c;
          const uint32_t take = work > 0 ? ((int64_t)work < budget ? work : (uint32_t)budget) : 1u;
          budget -= take;
          reserved += need;
          if (lane == 0) {
            const int j = nrun + took;
            sl.rq[j] = (uint32_t)(admit + k);
            sl.left[j] = work;   // updated after the iteration
            sl.dec[j] = take;    // scratch: tokens scheduled this iteration
            sl.kv[j] = c;
            sl.out[j] = o;
            sl.ptot[j] = p + o;
            sl.t_first[j] = 0.0;
            sl.arr[j] = a;
          }
          adm_tok += take;
          if (work > 0) adm_pf += take;
          if (take < work) adm_partial = true;
          adm_kv += c;
          adm_kvw += W ? min(c, W) : 0u;
          ++took;
        }
        nrun += took;
        admit += took;
        n_adm += took;
        if (blocked || took < 32) break;
      }
      if (nrun == 0) {  // head request can never fit the KV capacity
        status = DOOLY_ERR_INVALID_ARG;
        break;
      }
      if (wbase != admit) ld_wait(admit);  // prefetch the next waiting requests
      __syncwarp();
      // ---- 3. iteration features
      uint32_t kvs = 0, kvw = 0;
#pragma unroll kSimUnroll
      for (int j = lane; j < n_dec; j += 32) {
        const uint32_t k = sl.kv[j];
        kvs += k;
        kvw += W ? min(k, W) : 0u;
      }
      kvs = warp_sum_u32(kvs);
      kvw = warp_sum_u32(kvw);
      if (take_p > 0) {
        const uint32_t k = sl.kv[nrun0 - 1];
        kvs += k;
        kvw += W ? min(k, W) : 0u;
      }
      kvs += adm_kv;
      kvw += adm_kvw;
      const uint32_t num_toks = (uint32_t)n_dec + take_p + adm_tok;
      const uint32_t prefill = take_p + adm_pf;
      const uint32_t batch = (uint32_t)n_dec + (take_p > 0 ? 1u : 0u) + (uint32_t)n_adm;
      // ---- 4. window of exactly predictable iterations.  If every
      // request still running after this iteration is decoding (the tail
      // prefill and every admitted prompt complete now) and no admission can
      // happen before an arrival (no request waits) or before a finish (the
      // FCFS head is blocked by the batch or KV cap), the following iterations
      // have a known composition: slot j runs wr_j iterations from this one,
      // decoding with wb_j + u KV tokens at iteration u >= 1, and leaves after
      // its last token.  Lane u evaluates iteration u's whole op list (the same
      // entry arithmetic and in-order sum as the serial path); the clock then
      // commits them in order, stopping before the first iteration that starts
      // with an arrival due (no stop while the head is blocked: arrivals only
      // queue).  Finishes inside the window are stamped with the clock of their
      // last iteration, exactly as the event loop would.
      bool fin_any = false;
      uint64_t freed = 0;
      const bool waiting = admit < arrive;
      const bool hard = waiting && (nrun >= MB || blocked);
      const bool p_done = !has_p || take_p == sl.left[nrun0 - 1];
      int64_t wmax = 1;
      uint32_t wB = 0;
      if (p_done && !adm_partial && (!waiting || hard)) {
        uint32_t rmax = 0, rmin = 0xFFFFFFFFu;
        if (W == 0) {
          s_hc[wid][lane] = 0u;
          s_hk[wid][lane] = 0u;
          __syncwarp();
        }
#pragma unroll kSimUnroll
        for (int j = lane; j < nrun; j += 32) {
          uint32_t b, r;
          const uint32_t o = sl.out[j];
          if (j < n_dec) {  // decoding: out - dec tokens to go
            b = sl.kv[j];
            r = o - sl.dec[j];
          } else if (j < nrun0) {  // the tail prefill, completing in this iteration
            b = sl.kv[j] + take_p - 1u;
            r = o > 1u ? o : 1u;
          } else {  // admitted now: prefill completes now (or fully cached: first decode)
            const uint32_t c = sl.kv[j];
            b = sl.left[j] > 0u ? c + sl.dec[j] - 1u : c;
            r = o > 1u ? o : 1u;
          }
          sl.wb[j] = b;
          sl.wr[j] = r;
          rmax = max(rmax, r);
          rmin = min(rmin, r);
          wB += b;
          if (W == 0 && r < 32u) {
            atomicAdd(&s_hc[wid][r], 1u);
            atomicAdd(&s_hk[wid][r], b);
          }
        }
        rmax = __reduce_max_sync(0xFFFFFFFFu, rmax);
        rmin = __reduce_min_sync(0xFFFFFFFFu, rmin);
        wB = warp_sum_u32(wB);
        wmax = hard ? rmin : rmax;
        if (wmax > 32) wmax = 32;
        if (wmax > cfg.max_iterations - it) wmax = cfg.max_iterations - it;
        __syncwarp();
      }
      if (wmax >= 2) {
        // features of iteration u (lane u); iteration 0 is the one scheduled above
        uint32_t nt = num_toks, pf = prefill, bt = batch, ks = kvs, kw = kvw;
        const uint32_t u = (uint32_t)lane;
        uint32_t F = 0, K = 0;  // finished-before-u counts and KV sums (bins r <= u)
        if (W == 0) {
          F = s_hc[wid][lane];
          K = s_hk[wid][lane];
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t f2 = __shfl_up_sync(0xFFFFFFFFu, F, o);
            const uint32_t k2 = __shfl_up_sync(0xFFFFFFFFu, K, o);
            if (lane >= o) {
              F += f2;
              K += k2;
            }
          }
        }
        if (u > 0) {
          uint32_t nr = 0;
          ks = 0;
          kw = 0;
          if (W == 0) {
            nr = (uint32_t)nrun - F;
            ks = (wB - K) + u * nr;
          } else {
            for (int j = 0; j < nrun; ++j) {
              const uint32_t b = sl.wb[j] + u;
              if (sl.wr[j] > u) {
                ++nr;
                ks += b;
                kw += min(b, W);
              }
            }
          }
          nt = bt = nr;
          pf = 0;
        }
        bool bad = false;
        double lat = 0.0;
        if (ptab != nullptr) {
          // iteration 0 (any composition) by entries across lanes, as the serial path
          double w0 = 0.0, w1 = 0.0;
          if (lane < ops.n_ops)
            w0 = mul(s_ops.rep[lane], entry_value(ops, &s_ops, lane, num_toks, prefill, batch, kvs,
                                                  kvw, bad));
          if (lane + 32 < ops.n_ops)
            w1 = mul(s_ops.rep[lane + 32], entry_value(ops, &s_ops, lane + 32, num_toks, prefill,
                                                       batch, kvs, kvw, bad));
          double* sw0 = s_sum[wid];
          sw0[lane] = w0;
          sw0[lane + 32] = w1;
          __syncwarp();
          if (lane == 0) {
            int e = 0;
#pragma unroll 4
            for (; e + 2 <= ops.n_ops; e += 2) {
              const double2 v = *reinterpret_cast<const double2*>(sw0 + e);
              lat = add(lat, v.x);
              lat = add(lat, v.y);
            }
            if (e < ops.n_ops) lat = add(lat, sw0[e]);
          } else {
            // decode iteration u: table products, attention entries evaluated
            const double* prow = ptab + (size_t)min(nt, (uint32_t)MB) * ops.n_ops;
            for (int e = 0; e < ops.n_ops; ++e) {
              double v;
              if (s_ops.feat[e] == DOOLY_FEAT_ATTN) {
                bool cl;
                v = mul(s_ops.rep[e],
                        clamp_floor(eval_attn(s_ops.attn[e], 0u, bt, s_ops.wslot[e] ? kw : ks), cl));
              } else {
                v = prow[e];
              }
              lat = add(lat, v);
            }
          }
          __syncwarp();
        } else if (pv_base != nullptr) {
          lat = window_latency(ops, &s_ops, pv_base + (size_t)wid * ops.n_ops * 32, lane, nt, pf,
                               bt, ks, kw, bad);
          bad = bad && (int64_t)u < wmax;
        } else if ((int64_t)u < wmax) {
          for (int e = 0; e < ops.n_ops; ++e)
            lat = add(lat, mul(s_ops.rep[e], entry_value(ops, &s_ops, e, nt, pf, bt, ks, kw, bad)));
        }
        if (__any_sync(0xFFFFFFFFu, bad)) {
          status = DOOLY_ERR_UNKNOWN_SIGNATURE;
          break;
        }
        double* sw = s_sum[wid];
        sw[lane] = lat;
        __syncwarp();
        const double next_arr = __shfl_sync(0xFFFFFFFFu, win_arr, 0);
        int weff = 0;
        double myclk = 0.0;
        for (int v = 0; v < (int)wmax; ++v) {
          if (!hard && v > 0 && arrive < n && next_arr <= clock) break;  // admit it first
          clock = add(clock, sw[v]);
          if (v == lane) myclk = clock;
          ++weff;
        }
        __syncwarp();
        if (log_feat != nullptr && lane < weff && it + lane < log_cap) {
          const int64_t row = shard * log_cap + it + lane;
          uint32_t* lf = log_feat + row * DOOLY_IT_FEATS;
          lf[0] = nt;
          lf[1] = pf;
          lf[2] = bt;
          lf[3] = ks;
          lf[4] = kw;
          log_lat[row] = lat;
        }
        it += weff;
        const double clk0 = __shfl_sync(0xFFFFFFFFu, myclk, 0);
#pragma unroll kSimUnroll
        for (int j0 = 0; j0 < nrun; j0 += 32) {
          const int j = j0 + lane;
          const bool valid = j < nrun;
          const uint32_t r = valid ? sl.wr[j] : 1u;
          const uint32_t p = r < (uint32_t)weff ? r : (uint32_t)weff;  // iterations it ran
          const double clk_last = __shfl_sync(0xFFFFFFFFu, myclk, (int)p - 1);
          if (valid) {
            const bool newf = j >= n_dec;  // first token in iteration 0
            const uint32_t rq = sl.rq[j];
            const uint32_t out_n = sl.out[j];
            sl.kv[j] = sl.wb[j] + p;
            sl.dec[j] = (newf ? 0u : sl.dec[j]) + p;
            sl.left[j] = 0u;
            double tf = 0.0;
            if (newf) {
              tf = clk0;
              sl.t_first[j] = clk0;
              ttft[base + rq] = clk0 - sl.arr[j];
            } else {
              tf = sl.t_first[j];
            }
            if (r <= (uint32_t)weff) {
              tpot[base + rq] = out_n >= 2 ? __ddiv_rn(clk_last - tf, (double)(out_n - 1)) : nan64();
              freed += (uint64_t)sl.ptot[j] * kvb;
              sl.rq[j] = 0xFFFFFFFFu;  // tombstone
              fin_any = true;
            }
          }
        }
      } else {
      // ---- 4s. one iteration: fused gather-evaluate-reduce over the call graph
      // lanes evaluate their entries and the repeat products in parallel; the
      // in-order sum then only chains the adds (shuffles issued 4 at a time)
      bool bad = false;
      double w0 = 0.0, w1 = 0.0;
      if (lane < ops.n_ops)
        w0 = mul(s_ops.rep[lane],
                 entry_value(ops, &s_ops, lane, num_toks, prefill, batch, kvs, kvw, bad));
      if (lane + 32 < ops.n_ops)
        w1 = mul(s_ops.rep[lane + 32],
                 entry_value(ops, &s_ops, lane + 32, num_toks, prefill, batch, kvs, kvw, bad));
      // the products go through shared memory: every lane then reads them in
      // op-list order two at a time (broadcast LDS.128), so the in-order sum
      // costs one load per two adds instead of two 32-bit shuffles and a select
      // per entry
      double* sw = s_sum[wid];
      sw[lane] = w0;
      sw[lane + 32] = w1;
      __syncwarp();
      double lat = 0.0;
      int e = 0;
#pragma unroll 4
      for (; e + 2 <= ops.n_ops; e += 2) {
        const double2 v = *reinterpret_cast<const double2*>(sw + e);
        lat = add(lat, v.x);
        lat = add(lat, v.y);
      }
      if (e < ops.n_ops) lat = add(lat, sw[e]);
      if (__any_sync(0xFFFFFFFFu, bad)) {
        status = DOOLY_ERR_UNKNOWN_SIGNATURE;
        break;
      }
      clock = add(clock, lat);
      if (log_feat != nullptr && it < log_cap && lane == 0) {
        const int64_t row = shard * log_cap + it;
        uint32_t* lf = log_feat + row * DOOLY_IT_FEATS;
        lf[0] = num_toks;
        lf[1] = prefill;
        lf[2] = batch;
        lf[3] = kvs;
        lf[4] = kvw;
        log_lat[row] = lat;
      }
      ++it;
      // ---- 5. advance request state, stamp tokens, release finished reservations
      for (int j = lane; j < nrun; j += 32) {
        bool fin = false;
        const uint32_t r = sl.rq[j];
        const uint32_t out_n = sl.out[j];
        if (j < n_dec) {  // decode: one token
          sl.kv[j] += 1;
          const uint32_t d = sl.dec[j] + 1;
          sl.dec[j] = d;
          fin = d >= out_n;
        } else {
          const bool admitted = j >= nrun0;
          const uint32_t take = admitted ? sl.dec[j] : take_p;
          if (take > 0) {
            const uint32_t l = sl.left[j];
            if (l > 0) {  // prefill chunk
              sl.left[j] = l - take;
              sl.kv[j] += take;
              sl.dec[j] = 0;
              if (l == take) {  // last chunk: emits the first output token
                sl.dec[j] = 1;
                sl.t_first[j] = clock;
                ttft[base + r] = clock - sl.arr[j];
                fin = out_n <= 1;
              }
            } else {  // fully cached request admitted this iteration: first decode step
              sl.kv[j] += 1;
              sl.dec[j] = 1;
              sl.t_first[j] = clock;
              ttft[base + r] = clock - sl.arr[j];
              fin = out_n <= 1;
            }
          }
        }
        if (fin) {
          tpot[base + r] =
              out_n >= 2 ? __ddiv_rn(clock - sl.t_first[j], (double)(out_n - 1)) : nan64();
          freed += (uint64_t)sl.ptot[j] * kvb;
          sl.rq[j] = 0xFFFFFFFFu;  // tombstone
          fin_any = true;
        }
      }
      }
      if (__any_sync(0xFFFFFFFFu, fin_any)) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) freed += __shfl_xor_sync(0xFFFFFFFFu, freed, o);
        reserved -= freed;
        // stable in-place compaction, 32 slots at a time (reads precede writes
        // within a chunk and writes never reach the next chunk)
        int w = 0;
#pragma unroll kSimUnroll
        for (int j0 = 0; j0 < nrun; j0 += 32) {
          const int j = j0 + lane;
          const bool valid = j < nrun;
          uint32_t rq = 0xFFFFFFFFu, lf = 0, dc = 0, kv = 0, on = 0, pt = 0;
          double tf = 0.0, ar = 0.0;
          if (valid) {
            rq = sl.rq[j];
            lf = sl.left[j];
            dc = sl.dec[j];
            kv = sl.kv[j];
            on = sl.out[j];
            pt = sl.ptot[j];
            tf = sl.t_first[j];
            ar = sl.arr[j];
          }
          const bool keep = rq != 0xFFFFFFFFu;
          const uint32_t km = __ballot_sync(0xFFFFFFFFu, keep);
          __syncwarp();
          if (keep) {
            const int dst = w + __popc(km & ((1u << lane) - 1u));
            sl.rq[dst] = rq;
            sl.left[dst] = lf;
            sl.dec[dst] = dc;
            sl.kv[dst] = kv;
            sl.out[dst] = on;
            sl.ptot[dst] = pt;
            sl.t_first[dst] = tf;
            sl.arr[dst] = ar;
          }
          w += __popc(km);
          __syncwarp();
        }
        nrun = w;
      }
      __syncwarp();
    }
    if (lane == 0) {
#ifdef SIM_PASS_COUNT
      n_iter_out[shard] = passes;
#else
      n_iter_out[shard] = it;
#endif
      clock_out[shard] = clock;
      status_out[shard] = status;
    }
  }
}


cudaError_t launch_sim(const dooly_oplist* ops, const dooly_sched* cfg, const void* aff,
                       int64_t n_aff, const void* attn, int64_t n_attn, const double* arrival,
                       const uint32_t* prompt, const uint32_t* output, const uint32_t* cached,
                       const int64_t* shard_off, int64_t n_shards, double* ttft, double* tpot,
                       int64_t* n_iter, double* final_clock, int32_t* shard_status,
                       uint32_t* it_log_feat, double* it_log_lat, int64_t it_log_cap, void* ws,
                       size_t ws_bytes, cudaStream_t stream, int n_sm) {
  (void)n_aff;
  (void)n_attn;
  (void)ws;
  (void)ws_bytes;
  (void)n_sm;
  if (n_shards == 0) return cudaSuccess;
  size_t smem = (size_t)SIM_WARPS * cfg->max_batch * kSlotBytes;
  // the window's product columns (n_ops x 32 doubles per warp) when they fit beside the slots
  const size_t pv = (size_t)SIM_WARPS * ops->n_ops * 32 * sizeof(double);
  int dev = 0, optin = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  cudaFuncAttributes fa;
  e = cudaFuncGetAttributes(&fa, sim_run_kernel);
  if (e != cudaSuccess) return e;
  // the decode-product table (one per CTA) when it fits, else the product columns
  const size_t pt = (size_t)(cfg->max_batch + 1) * ops->n_ops * sizeof(double);
  const char* pvenv = getenv("DOOLY_SIM_PV");
  const int want = pvenv != nullptr ? atoi(pvenv) : 2;
  int use_pv = 0;
  if (want >= 2 && smem + pt + fa.sharedSizeBytes <= (size_t)optin) {
    use_pv = 2;
    smem += pt;
  } else if (want >= 1 && smem + pv + fa.sharedSizeBytes <= (size_t)optin) {
    use_pv = 1;
    smem += pv;
  }
  e = cudaFuncSetAttribute(sim_run_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t blocks = (n_shards + SIM_WARPS - 1) / SIM_WARPS;
  sim_run_kernel<<<(unsigned)blocks, SIM_WARPS * 32, smem, stream>>>(
      *ops, *cfg, aff, attn, arrival, prompt, output, cached, shard_off, n_shards, ttft, tpot,
      n_iter, final_clock, shard_status, it_log_feat, it_log_lat, it_log_cap, use_pv);
  return cudaGetLastError();
}

}  // namespace dooly

// ===================================================================
// dooly_sim_eval: host-scheduled iterations (an external simulator's own
// scheduler, "drop-in profiling backend") evaluated on the
// device.  iter_eval gives it_lat; then one warp per shard scans
// clock[i] = max(clock[i-1], it_start[i]) + it_lat[i] sequentially (the same
// f64 operation order as the event loop: an idle replica
// jumps to the next arrival, else iterations run back to back); then one
// thread per request reads its first/last-token clocks.
namespace dooly {

// One warp per shard.  The recurrence is inherently sequential (the same f64
// operation order as the event loop), so lane 0 runs it over a 256-iteration
// chunk staged in shared memory by the whole warp (coalesced loads of it_lat /
// it_start, the next chunk's loads issued before the scan), then the warp
// writes the chunk's clocks back coalesced.
constexpr int kClockChunk = 256;
constexpr int kClockWarps = 4;

__global__ void __launch_bounds__(32 * kClockWarps) sim_clock_kernel(
    const double* __restrict__ it_lat, const double* __restrict__ it_start,
    const int64_t* __restrict__ it_off, int64_t n_shards, int64_t n_it,
    double* __restrict__ clock) {
  __shared__ double sl[kClockWarps][kClockChunk], ss[kClockWarps][kClockChunk];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= n_shards) return;
  const int64_t b = it_off ? it_off[w] : 0, e = it_off ? it_off[w + 1] : n_it;
  double* L = sl[wid];
  double* S = ss[wid];
  constexpr int PER = kClockChunk / 32;
  double nl[PER], ns[PER];
  auto fetch = [&](int64_t i0) {
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int64_t i = i0 + k * 32 + lane;
      nl[k] = i < e ? it_lat[i] : 0.0;
      ns[k] = (i < e && it_start) ? it_start[i] : 0.0;
    }
  };
  double c = 0.0;
  fetch(b);
  for (int64_t i0 = b; i0 < e; i0 += kClockChunk) {
    bool jump = false;  // an idle jump target anywhere in this chunk
#pragma unroll
    for (int k = 0; k < PER; ++k) jump |= __double_as_longlong(ns[k]) != 0ll;
    jump = __any_sync(0xFFFFFFFFu, jump);
    const int m = (int)min((int64_t)kClockChunk, e - i0);
    if (!jump) {
      // busy chunk (it_start == 0 throughout, the common case): iteration
      // k*32 + l sits in lane l's cur[k]; every lane runs the same add chain
      // over shuffled values (no shared memory, the shuffles are independent
      // of the chain) and lane l keeps the clocks of its own iterations.
      // Past the end of the shard the values are 0.0: adding them leaves the
      // clock as is, and they are not stored.
      double cur[PER], out[PER];
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        cur[k] = nl[k];
        out[k] = 0.0;
      }
      if (i0 + kClockChunk < e) fetch(i0 + kClockChunk);   // next chunk in flight
#pragma unroll
      for (int k = 0; k < PER; ++k) {
#pragma unroll
        for (int l = 0; l < 32; ++l) {
          c = __dadd_rn(c, __shfl_sync(0xFFFFFFFFu, cur[k], l));
          out[k] = lane == l ? c : out[k];
        }
      }
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int64_t i = i0 + k * 32 + lane;
        if (i < e) clock[i] = out[k];
      }
      continue;
    }
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      L[k * 32 + lane] = nl[k];
      S[k * 32 + lane] = ns[k];
    }
    __syncwarp();
    if (i0 + kClockChunk < e) fetch(i0 + kClockChunk);   // next chunk in flight during the scan
    if (lane == 0) {
      // the max with an idle jump target on a nonzero start
#pragma unroll 8
      for (int j = 0; j < m; ++j) {
        const double sj = S[j];
        if (__double_as_longlong(sj) != 0ll && c < sj) c = sj;
        c = __dadd_rn(c, L[j]);
        L[j] = c;
      }
    }
    c = __shfl_sync(0xFFFFFFFFu, c, 0);
    __syncwarp();
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int64_t i = i0 + k * 32 + lane;
      if (i < e) clock[i] = L[k * 32 + lane];
    }
    __syncwarp();
  }
}

__global__ void __launch_bounds__(256) sim_request_kernel(
    const double* __restrict__ clock, int64_t n_it, const double* __restrict__ arrival,
    const uint32_t* __restrict__ first_it, const uint32_t* __restrict__ last_it,
    const uint32_t* __restrict__ out_tok, int64_t n_req, double* __restrict__ ttft,
    double* __restrict__ tpot, int64_t* __restrict__ err_first) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_req;
       r += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t f = first_it[r], l = last_it[r], o = out_tok[r];
    double t1 = nan64(), t2 = nan64();
    if (f != 0xFFFFFFFFu) {
      if (f >= n_it || (l != 0xFFFFFFFFu && (l >= n_it || l < f))) {
        if (err_first)
          atomicMin(reinterpret_cast<unsigned long long*>(err_first), (unsigned long long)r);
      } else {
        const double cf = clock[f];
        t1 = __dsub_rn(cf, arrival[r]);
        if (o >= 2 && l != 0xFFFFFFFFu) t2 = __ddiv_rn(__dsub_rn(clock[l], cf), (double)(o - 1));
      }
    }
    ttft[r] = t1;
    tpot[r] = t2;
  }
}

cudaError_t launch_sim_eval(const double* it_lat, const double* it_start, const int64_t* it_off,
                            int64_t n_shards, int64_t n_it, double* clock, const double* arrival,
                            const uint32_t* first_it, const uint32_t* last_it,
                            const uint32_t* out_tok, int64_t n_req, double* ttft, double* tpot,
                            int64_t* err_first, cudaStream_t stream, int n_sm,
                            int64_t* launches) {
  if (n_it > 0 && n_shards > 0) {
    const int64_t blocks = (n_shards + kClockWarps - 1) / kClockWarps;
    sim_clock_kernel<<<(unsigned)blocks, 32 * kClockWarps, 0, stream>>>(it_lat, it_start, it_off,
                                                                        n_shards, n_it, clock);
    *launches += 1;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (n_req > 0) {
    int64_t blocks = (n_req + 255) / 256;
    if (blocks > (int64_t)n_sm * 8) blocks = (int64_t)n_sm * 8;
    sim_request_kernel<<<(unsigned)blocks, 256, 0, stream>>>(clock, n_it, arrival, first_it,
                                                             last_it, out_tok, n_req, ttft, tpot,
                                                             err_first);
    *launches += 1;
  }
  return cudaGetLastError();
}

}  // namespace dooly
