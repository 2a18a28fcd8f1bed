/*
 * niyama.h — C ABI of the B200-native hybrid-batch paged-attention path of
 * Niyama (arXiv 2503.22562).  Library: paper_2503_22562_b200/libniyama.so
 *
 * Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n,
 * §8 = SURVEY.md §8 (the hot-path scope table), Rn = DESIGN.md reading n.
 *
 * What the path computes.  Each serving iteration Niyama builds ONE hybrid
 * batch: the decode step of every running request plus a prefill chunk
 * (§3.1 steps ④-⑥: "A lightweight predictor is then used to estimate
 * the latency of the batch ... A mixed batch of prefill and decode tokens is
 * constructed ... dispatched to the execution engine on the GPU").  Attention
 * of that batch over a block-table KV cache (vLLM PagedAttention, P:319
 * §3.6) is the data-parallel hot path.  For batch row r (visible keys n_r)
 * and query head h (kv head h / (Hq/Hkv), R7):
 *     O[h][r] = softmax(scale * q_{r,h} K^T) V,  LSE[h][r] = ln sum exp(...)
 * with causal visibility (prefill row at position p sees keys [0, p]; a
 * decode row sees its whole context, R4).  §8(a) rows a1-a8 map to:
 *   a1 niyama_min_slack + niyama_max_feasible_chunk      (host, fp64)
 *   a2 niyama_plan_create                                (host planner)
 *   a3 niyama_kv_append                                  (scatter kernel)
 *   a4-a6 niyama_hybrid_attention                        (ONE fused launch)
 *   a3-a6 niyama_append_attention                        (append + attention, ONE launch)
 *   a7 niyama_comm_init + niyama_allgather_heads         (NCCL over NVLink)
 *   §8(f)2 niyama_gather_create + niyama_attention_gather (all-gather fused into the launch)
 *   a8 niyama_predictor_fit + niyama_predict_iter_time   (host, fp64)
 *   §8(f)1 niyama_sched_*: QoS scheduler core            (host)
 *
 * Conventions (all calls):
 *  - Every call returns niyama_status unless noted; on error the message is
 *    available from niyama_last_error() (thread-local, valid until the next
 *    call on the same thread).  Validation happens before any side effect or
 *    launch; the API never aborts and takes no locks.  One niyama_kv per
 *    host thread / stream (single-threaded per replica).
 *  - "device" pointers are CUDA global-memory pointers on cfg.device;
 *    "host" pointers are ordinary host memory.  All device work is enqueued
 *    on the caller's stream and is asynchronous; a plan must outlive every
 *    launch that uses it (destroy is stream-ordered).
 *  - Tensors are dense row-major, no padding.  bf16 values are raw IEEE
 *    bfloat16; f32 values are IEEE binary32.
 *  - There is no CPU fallback: with cfg.device = NIYAMA_DEVICE_NONE the
 *    library keeps only host bookkeeping (planner tests) and every call that
 *    would touch the GPU returns NIYAMA_EUNSUPPORTED.
 */
#ifndef NIYAMA_H_
#define NIYAMA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* niyama_stream; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
  NIYAMA_OK = 0,
  NIYAMA_EINVAL = 1,       /* malformed argument or descriptor (names the field) */
  NIYAMA_ENOBLOCKS = 2,    /* KV pool exhausted; nothing was reserved (all-or-nothing) */
  NIYAMA_ENOSEQ = 3,       /* decode / release / gather of an unknown sequence */
  NIYAMA_ESTATE = 4,       /* cached length != prefill offset, or != decode ctx-1 (R4) */
  NIYAMA_ECUDA = 5,        /* CUDA runtime/launch failure (message has cudaGetErrorString) */
  NIYAMA_ENCCL = 6,        /* NCCL failure */
  NIYAMA_EUNSUPPORTED = 7  /* shape/dtype not built, or no device (NIYAMA_DEVICE_NONE) */
} niyama_status;

const char* niyama_last_error(void);
const char* niyama_version(void);

#define NIYAMA_DEVICE_NONE (-1)

/* Device use: every call that touches the GPU runs on cfg.device and restores the
 * calling thread's current device before returning.
 *
 * Failure and recovery: a kernel that detects a lost completion (a watchdog of ~2^26
 * polls in the in-launch merge / append wait) executes a trap.  A trap, like any
 * kernel fault, is a sticky CUDA context error: every later call on the device returns
 * NIYAMA_ECUDA, and the context (and with it the pool, plans and communicator) cannot
 * be reused — the process must destroy its objects and restart (the serving layer
 * re-plans the iteration from its own request state; KV bytes are lost with the
 * context).  A launch that fails to START (configuration error, returned as ECUDA)
 * changes nothing: the plan's launch count and queues are untouched and the call may
 * be retried.  A plan's launches must be ordered on one stream (or explicitly
 * ordered): they share the plan's work queues and completion counters. */

typedef enum { NIYAMA_BF16 = 0, NIYAMA_F32 = 1 } niyama_dtype;

/* KV-cache configuration.  Heads are GLOBAL counts; with world_size G the
 * library on `rank` owns kv heads [rank*Hkv/G, (rank+1)*Hkv/G) and query
 * heads [rank*Hq/G, (rank+1)*Hq/G) (GQA groups stay whole, §8e
 * tensor parallelism).  Supported (anything else is EUNSUPPORTED at create):
 * bf16 head_dim 128; f32 head_dim 32, 64, 96 or 128; Hq/Hkv a power of two
 * <= 8; block_size in {16, 32, 64, 128} (R9: default 16). */
typedef struct {
  int32_t num_layers;
  int32_t num_q_heads;
  int32_t num_kv_heads;
  int32_t head_dim;
  int32_t block_size;
  int32_t num_blocks;   /* pool capacity in blocks (each block holds block_size tokens of every local kv head) */
  niyama_dtype dtype;   /* stored type of K/V/Q/O */
  int32_t world_size;   /* >= 1 */
  int32_t rank;         /* 0 <= rank < world_size */
  int32_t device;       /* CUDA ordinal, or NIYAMA_DEVICE_NONE (host bookkeeping only) */
} niyama_kv_config;

typedef struct niyama_kv niyama_kv;
typedef struct niyama_plan niyama_plan;

/* Create the pool.  The library allocates and OWNS num_layers*2*num_blocks*
 * (Hkv/G)*block_size*head_dim elements of device memory (zero-filled) plus
 * the block tables.  Errors: EINVAL (shape), EUNSUPPORTED, ECUDA (OOM). */
niyama_status niyama_kv_create(const niyama_kv_config* cfg, niyama_kv** out);
void niyama_kv_destroy(niyama_kv* kv); /* synchronises the device; NULL is a no-op.  Destroy every plan of
                                          * this kv first: their buffers live in its memory pool. */

/* Request finished (P:205 ⑦, §8 a13 feedback): free its blocks (they become
 * the smallest-free-id candidates again, R9).  ENOSEQ if unknown. */
niyama_status niyama_kv_release(niyama_kv* kv, int64_t seq_id);
/* Roll a sequence back to its first new_len tokens (new_len <= cached
 * length): blocks beyond ceil(new_len/B) return to the free set (R9).  Host
 * bookkeeping only; KV bytes are not touched (stream order keeps in-flight
 * launches valid: a later plan that re-reserves a block is ordered after
 * them on the same stream).  Used for iteration replay and rollback. */
niyama_status niyama_kv_truncate(niyama_kv* kv, int64_t seq_id, int32_t new_len);
/* Host read of a sequence's block table: n = number of blocks; copies
 * min(n, cap) ids to out (host).  ENOSEQ if unknown. */
niyama_status niyama_kv_block_table(const niyama_kv* kv, int64_t seq_id, int32_t* out, int32_t cap, int32_t* n);
niyama_status niyama_kv_seq_len(const niyama_kv* kv, int64_t seq_id, int32_t* len);
niyama_status niyama_kv_num_free(const niyama_kv* kv, int32_t* n);
/* Test read-back: logical K and V of positions [0, len) of seq in layer, as
 * dense [len][Hkv_loc][head_dim] in the stored dtype, to DEVICE buffers
 * k_out, v_out.  EINVAL if len > cached length. */
niyama_status niyama_kv_gather(niyama_kv* kv, int32_t layer, int64_t seq_id, int32_t len, void* k_out,
                               void* v_out, niyama_stream stream);

/* One iteration's hybrid batch (P:205 ⑤; D2 in SURVEY §2.3).  HOST pointers,
 * copied during niyama_plan_create (caller may free afterwards).
 * Rows of the batch: prefill slice i contributes prefill_len[i] rows at
 * positions prefill_offset[i] .. +len-1 (in slice order), then one row per
 * decode j at position decode_ctx[j]-1 (R6).  A slice of an unknown seq
 * with offset 0 creates the sequence (len 0 is allowed and just registers
 * it).  decode_ctx counts the keys visible after appending the new token
 * (R4).  A seq id may appear at most once per batch.  tier[i] (i over
 * slices then decodes; may be NULL) is the request's QoS tier, 0 = strictest
 * (Table 3); it only orders work inside the launch and never changes
 * any result bit (R13). */
typedef struct {
  int32_t num_prefill;
  const int64_t* prefill_seq;
  const int32_t* prefill_offset;
  const int32_t* prefill_len;
  int32_t num_decode;
  const int64_t* decode_seq;
  const int32_t* decode_ctx;
  const uint8_t* tier;
} niyama_batch_desc;

/* a2 — plan an iteration: validate (EINVAL/ENOSEQ/ESTATE), reserve blocks
 * (smallest free ids, descriptor order, all-or-nothing → ENOBLOCKS, R9),
 * advance the cached lengths, and build the device work list (prefill tiles
 * and split-KV decode units, longest first) with ONE async H2D on `stream`.
 * The plan is reused by every layer's append/attention of the iteration. */
niyama_status niyama_plan_create(niyama_kv* kv, const niyama_batch_desc* desc, niyama_stream stream,
                                 niyama_plan** out);
void niyama_plan_destroy(niyama_plan* plan); /* stream-ordered free on the plan's stream; before the plan's
                                               * niyama_kv is destroyed */
/* Undo the plan's host bookkeeping: every sequence of the batch returns to its
 * length before niyama_plan_create (sequences the plan created are removed);
 * blocks past the old lengths are freed (R9).  An entry applies only to the
 * sequence the plan saw (same id and creation generation): a sequence released
 * meanwhile — or released and re-created under the same id — is left alone.
 * Every entry is validated before anything changes (ESTATE if a sequence is now
 * shorter than before the plan; nothing rolled back).  The plan's device buffers
 * stay valid for launches already enqueued.  Used to abort or replay an iteration. */
niyama_status niyama_plan_rollback(niyama_kv* kv, niyama_plan* plan);

typedef struct {
  int32_t num_rows;           /* T = sum prefill_len + num_decode */
  int32_t num_prefill_rows;
  int32_t num_decode;
  int32_t num_prefill_tiles;  /* 128-row (packed GQA) x 128-key tcgen05 tiles */
  int32_t num_decode_units;   /* (decode row, kv head, key split) items */
  int32_t split_len;          /* decode split length in tokens (batch-level choice) */
  int32_t rows_per_tile;      /* 128 / (Hq/Hkv) chunk rows per prefill tile */
  int32_t prefill_ctas;       /* bf16 launch: CTAs that take prefill tiles before decode units
                                 (work-proportional split); 0 if no tiles */
  int64_t sum_ctx;            /* sum of decode ctx */
} niyama_plan_info;
niyama_status niyama_plan_get_info(const niyama_plan* plan, niyama_plan_info* out);
/* Host copy of the slot map: row r's new K/V goes to (block_out[r], slot_out[r]). */
niyama_status niyama_plan_slots(const niyama_plan* plan, int32_t* block_out, int32_t* slot_out, int32_t cap);

/* a3 — scatter the batch's new K/V rows into the pool (bit copy, no dtype
 * conversion): pool[table[s][p/B]][h][p%B] = K_new[row][h].  k_new, v_new:
 * DEVICE [T][Hkv_loc][head_dim]. */
niyama_status niyama_kv_append(niyama_kv* kv, const niyama_plan* plan, int32_t layer, const void* k_new,
                               const void* v_new, niyama_stream stream);

/* a4-a6 — ONE launch: causal prefill-chunk tiles (tcgen05/TMEM, bf16) and
 * split-KV decode units (HBM-bound, mma.sync) with the log-sum-exp merge of
 * a row's splits done in-launch by its last split (merge order = split
 * order, so results are bitwise deterministic).
 *   q   DEVICE [T][Hq_loc][head_dim]   (post-RoPE, R8)
 *   o   DEVICE [Hq_loc][T][head_dim]   (head-major so the all-gather needs no transpose)
 *   lse DEVICE [Hq_loc][T] f32 natural-log LSE (R11), or NULL
 *   softmax_scale <= 0 selects 1/sqrt(head_dim).
 * Append must have been enqueued before for the same layer and plan.
 * T = 0 is a no-op. */
niyama_status niyama_hybrid_attention(niyama_kv* kv, const niyama_plan* plan, int32_t layer, const void* q,
                                      void* o, float* lse, float softmax_scale, niyama_stream stream);

/* a3 + a4-a6 in ONE launch: the result of niyama_kv_append followed by
 * niyama_hybrid_attention (same arguments, same layouts, same outputs).  bf16:
 * the attention launch scatters k_new / v_new into the pool itself before any
 * tile or decode unit reads it (CTAs claim append pieces from a queue, every
 * CTA waits for the completion count, which needs no co-residency because all
 * pieces are claimed by running CTAs) — one launch per layer instead of two.
 * f32: the two launches.  Errors as the two calls. */
niyama_status niyama_append_attention(niyama_kv* kv, const niyama_plan* plan, int32_t layer, const void* k_new,
                                      const void* v_new, const void* q, void* o, float* lse, float softmax_scale,
                                      niyama_stream stream);

/* Diagnostics: when device_buf (DEVICE, int64, >= 160*8 + 10*64 entries,
 * zeroed by the caller) is non-NULL every later niyama_hybrid_attention
 * writes, per CTA c at [8c..8c+5]: globaltimer ns at start, end of its
 * prefill tiles, exit, #prefill tiles, end of its decode units, grid barrier
 * passed; and at [1280 + 64*role + j] CTA 0's clock64 when key tile j of its
 * first prefill tile passed role's step (0 K issue, 1 V issue, 2 QK issue,
 * 3 PV issue, 4 S ready, 5 row max done, 6 P written, 7 rescale done, 8-9 P half
 * written).  NULL = off (default). */
niyama_status niyama_debug_trace(niyama_kv* kv, int64_t* device_buf);

/* Launch tuning (explicit, per kv; default = the planner's own choices).  Used by the
 * measurement tools; the predictor sees the same values through niyama_predictor_bind.
 *   prefill_ctas      0 = work-proportional CTA split; n > 0 = at most n CTAs take
 *                     prefill tiles first
 *   split_len         0 = decode split length from batch totals; else a multiple of 16
 *   tail_div, tail_min  a row's last piece is cut into min(q, max(tail_min, q/tail_div))
 *                     tokens (defaults NIYAMA_TAIL_DIV, NIYAMA_TAIL_MIN)
 *   grid_cap          0 = grid from the plan; n > 0 = at most n CTAs (diagnostics)
 *   plan_copy_stream  1 = plans upload on the library's copy stream (default), 0 = on
 *                     the caller's stream
 *   prefill_split     1 = split-K of prefill q tiles when they are fewer than their CTAs (key
 *                     parts on different CTAs, merged by the last part; parity-tested, measured
 *                     slower: DESIGN.md 6.1), 0 = never split (default)
 *   decode_path       bf16 decode units: 0 = auto (default: 2 when g > 4, else 3), 1 = one
 *                     tensor-core (tcgen05) pipeline per CTA over 128-token steps (measured
 *                     slower: DESIGN.md 6.1), 2 = producer warps: warps 8-11 claim units and
 *                     issue the stage copies of two compute warps each (warps 0-7), 3 = every
 *                     decode warp is its own loader (12 warps at g <= 4, 8 at g = 8).  All
 *                     paths give the same results within bf16 rounding; 0, 2 and 3 are bitwise
 *                     identical (same units, same per-unit arithmetic)
 *   prefill_pairs     0 = auto (default: pairs when g > 4), 1 = prefill q tiles run in CTA
 *                     pairs (clusters of 2): the two q tiles (qt, qt - 1) of a kv head share
 *                     every K/V step, each CTA issuing half of the step's bulk copies multicast
 *                     into both (half the TMA issue and L2 reads per SM; bitwise identical
 *                     results); 2 = one q tile per CTA.  Ignored with prefill_split
 * A changed tuning applies to plans created afterwards (split, CTA split) and to
 * launches issued afterwards (grid cap). */
typedef struct {
  int32_t prefill_ctas;
  int32_t split_len;
  int32_t tail_div;
  int32_t tail_min;
  int32_t grid_cap;
  int32_t plan_copy_stream;
  int32_t decode_path;
  int32_t prefill_split;
  int32_t prefill_pairs;
} niyama_tuning;
niyama_status niyama_kv_get_tuning(const niyama_kv* kv, niyama_tuning* out);
niyama_status niyama_kv_set_tuning(niyama_kv* kv, const niyama_tuning* t); /* EINVAL on out-of-range fields */

/* a7 — head sharding across the GPUs of one node (§8e).  comm_init creates
 * the library's own NCCL communicator from a 128-byte ncclUniqueId produced
 * by rank 0 and broadcast by the caller (world/rank from the config).
 * allgather_heads (ncclAllGather, issued at every world size — at 1 it is NCCL's
 * in-place copy; EINVAL before comm_init) gathers every rank's [Hq/G][T][d] slice into o_full
 * [Hq][T][d] IN PLACE (this rank's slice must already sit at
 * o_full + rank*(Hq/G)*T*d) and likewise lse_full [Hq][T] if non-NULL. */
niyama_status niyama_comm_init(niyama_kv* kv, const void* nccl_unique_id);
niyama_status niyama_get_unique_id(void* out128); /* ncclGetUniqueId, for rank 0 */
niyama_status niyama_allgather_heads(niyama_kv* kv, const niyama_plan* plan, void* o_full, float* lse_full,
                                     niyama_stream stream);

/* §8(f)2 — the head all-gather fused into the attention launch (
 * the exchange is a7's, P:319 TP -> head sharding, §8e).  Instead of a separate
 * collective after the kernel, every O row (and LSE value) the launch produces is
 * stored straight into the output window of EVERY rank (NVLink load/store through
 * NCCL symmetric memory: ncclMemAlloc + ncclCommWindowRegister, peer addresses from
 * the window's LSA mapping), and the launch's last CTA runs a flag barrier with the
 * other ranks' launches, so when the kernel completes on rank r its window holds all
 * G ranks' heads.  bf16 pools only.
 *
 * niyama_gather_create (COLLECTIVE over kv's communicator: every rank calls it, after
 * niyama_comm_init, with the same max_rows) allocates one window holding two output
 * buffers of o_full [Hq][max_rows][d] bf16 + lse_full [Hq][max_rows] f32 (Hq = all
 * ranks' heads) and the barrier flags.  EUNSUPPORTED if the NCCL build or the system
 * gives no symmetric memory (then use niyama_allgather_heads); EINVAL before
 * comm_init, on an f32 pool or max_rows <= 0.  niyama_gather_destroy is collective too
 * (stream-ordered: call it after the last launch's stream work completed).
 *
 * niyama_attention_gather = niyama_append_attention (k_new, v_new may be NULL: no
 * append) whose outputs go to the window: on return *o_full / *lse_full (DEVICE, this
 * rank's mapping) point at the buffer the launch fills, head-major [Hq][T][d] / [Hq][T]
 * exactly as niyama_allgather_heads leaves them (rank r's heads at r*(Hq/G)).  The two
 * buffers alternate per call, so a buffer is rewritten only by the call after next;
 * a rank must finish reading the outputs of call n (stream-ordered work is enough)
 * before it issues call n + 1, and every rank must issue the same sequence of calls
 * (the barrier matches them by count; a rank that never arrives makes the others trap
 * after ~30 s instead of hanging).  plan->T <= max_rows (else EINVAL). */
typedef struct niyama_gather niyama_gather;
niyama_status niyama_gather_create(niyama_kv* kv, int32_t max_rows, niyama_gather** out);
niyama_status niyama_gather_destroy(niyama_gather* g);
niyama_status niyama_attention_gather(niyama_kv* kv, const niyama_plan* plan, int32_t layer, const void* k_new,
                                      const void* v_new, const void* q, niyama_gather* g, float softmax_scale,
                                      void** o_full, float** lse_full, niyama_stream stream);
/* Test support for the same protocol without NVLink peers: n library instances of ONE
 * process on ONE device, kvs[r] = rank r of world n (bf16, same shape), get n windows in
 * ordinary device memory (cudaMalloc) cross-linked as each other's peers; the ranks'
 * niyama_attention_gather launches must then run CONCURRENTLY (one stream per rank) — a
 * launch's last CTA waits for the others'.  Destroy each with niyama_gather_destroy. */
niyama_status niyama_debug_gather_group(niyama_kv* const* kvs, int32_t n, int32_t max_rows, niyama_gather** outs);

/* a8 — iteration-time predictor (P:205 ④ "A lightweight predictor is then used
 * to estimate the latency of the batch"; reading R16).  The paper's
 * predictor is a random forest on profiles; this one is an EVENT MODEL of the
 * fused launch fitted to measured launch times, evaluated on this
 * rank's shape.  The launch-shaping rules are the planner's own (one definition,
 * csrc/internal.h), so the model sees the launch the kernel runs:
 *
 *  1. Prefill work queue: slices (o, c > 0) sorted by o + c descending (stable);
 *     per slice the q tiles from last to first (qt = nqt-1 .. 0, nqt = ceil(c/R),
 *     R = 128 / (Hq/Hkv)), each repeated Hkv times, with nk = ceil((o + min(c,
 *     (qt+1) R)) / 128) key steps, cut into the planner's split-K parts P (the
 *     target floor(prefill CTAs / q tiles) <= 16, per slice at most its shortest
 *     tile's steps / 4): part i has floor((i+1) nk / P) - floor(i nk / P) steps.
 *  2. Decode unit queue: split length q from (sum ctx, max ctx) as the planner;
 *     rows by ctx descending contribute ceil(L/q) - 1 full pieces of q keys
 *     (x Hkv units each), then every row's last L - n_f q keys cut into pieces of
 *     min(q, max(tail_min, q / tail_div)) keys, all such pieces longest first
 *     (x Hkv).  A unit of k keys streams k * d * 2 * elt bytes.
 *  3. grid and prefill CTAs n_p: the planner's CTA split (niyama_plan_info).
 *  4. Prefill: a step lasts tau = tau0 + tau_p n_p/NIYAMA_PRED_SMS
 *     + tau_d (grid - n_p)/grid (the last term only with decode units: HBM
 *     contention from the decode CTAs); each tile in queue order goes to the
 *     prefill CTA that frees first and occupies it (s + sigma) tau seconds.
 *  5. Decode: grid - n_p CTAs' warps (12 per CTA when Hq/Hkv <= 4, else 8) are
 *     free at 0, each prefill CTA's warps when its last tile ends; each unit in
 *     queue order goes to the warp that frees first (at time a) and occupies it
 *     u0 + bytes / min(r_w, BW / W(a)) seconds, W(a) = warps streaming by a.
 *  6. T_sim = the later of the last tile and the last unit to end;
 *     t_hat = theta[0] + theta[1] (c + D) + theta[2] D + theta[3] sum ctx
 *             + theta[4] units + theta[5] T_sim   (c = prefill rows, D = decodes).
 * Parameters (NIYAMA_NUM_PARAMS doubles): theta[0..5] >= 0 (linear part);
 * theta[6..12] = tau0 (s), tau_p (s), tau_d (s), sigma (steps), r_w (B/s),
 * u0 (s), BW (B/s), all > 0.  SPEC's affine model is the special case
 * theta[0..5] = (c0, c1, 0, c2, 0, 0).
 * Fit (niyama_predictor_fit_batches): Nelder-Mead over the logarithms of
 * theta[6..12] (then once more from its best vertex); for each candidate, the
 * simulations of all samples and theta[0..4] >= 0 by non-negative least squares on
 * relative residuals with theta[5] = 1; the objective is the sum of squared
 * relative errors.  Deterministic. */
#define NIYAMA_PRED_SMS 148
#define NIYAMA_TAIL_DIV 4
#define NIYAMA_TAIL_MIN 256
/* CTA split: one 128-key prefill step weighs as much CTA time as this many bytes of decode
 * KV (recalibrated late in round 2 on the faster kernel, tools/cap_sweep.py: the best fixed
 * prefill-CTA counts of 15 L8B shapes imply 95-125 KB; round 1 used 160 KB, which gave
 * config 2 60 prefill CTAs where 48 measured 2 % faster and c1024/o1024/D64 10 % slower
 * than its best). */
#define NIYAMA_STEP_BYTES 115e3
/* CTA split: decode KV bytes weigh this much more when g = Hq/Hkv > 4 (the launch then
 * streams decode with 8 compute warps per CTA instead of 12, so a CTA moves fewer bytes per
 * unit time; config 4: 858 us at the rule's 82-84 CTAs, 861 at 80, 866 at 88, 963 at 72,
 * tools/cap_sweep_l70b.py). */
#define NIYAMA_WIDE_GROUP_DECODE_WEIGHT 1.25
#define NIYAMA_TILE_SETUP_STEPS 2
#define NIYAMA_NUM_PARAMS 16

typedef struct {
  int32_t chunk_len;    /* prefill rows of the (single) slice, 0 if none */
  int32_t chunk_offset;
  int32_t num_decode;
  int64_t sum_ctx;      /* sum of decode ctx (>= num_decode); the model spreads it evenly over the decodes */
  double seconds;       /* measured launch time (> 0) */
} niyama_sample;
typedef struct niyama_predictor niyama_predictor;
typedef struct {
  const double* start;  /* NIYAMA_NUM_PARAMS starting values (only theta[6..12] are used), or NULL = defaults */
  int32_t max_evals;    /* Nelder-Mead objective evaluations (0 = 1200, plus half as many on the restart) */
  int32_t subsample;    /* Nelder-Mead on every k-th sample (0/1 = all); the final linear fit uses all */
} niyama_fit_options;

/* Fit on measured launches: batch i (its slices and decode contexts; tiers ignored) took
 * seconds[i] > 0.  opt may be NULL.  Host pointers; EINVAL on an invalid sample. */
niyama_status niyama_predictor_fit_batches(const niyama_kv_config* shape, const niyama_batch_desc* batches,
                                           const double* seconds, int32_t n, const niyama_fit_options* opt,
                                           niyama_predictor** out);
/* The same fit on summary samples (each a single slice + decodes with sum ctx spread evenly). */
niyama_status niyama_predictor_fit(const niyama_kv_config* shape, const niyama_sample* samples, int32_t n,
                                   niyama_predictor** out);
niyama_status niyama_predictor_from_params(const niyama_kv_config* shape, const double* theta,
                                           niyama_predictor** out); /* theta[0..5] >= 0, theta[6..12] > 0 */
niyama_status niyama_predictor_params(const niyama_predictor* p, double* theta_out);
/* Seconds for the batch (slices and decodes of desc; tiers ignored); < 0 on invalid input. */
double niyama_predict_iter_time(const niyama_predictor* p, const niyama_batch_desc* desc);
typedef struct {
  int32_t grid, prefill_ctas;   /* step 3 */
  int32_t split_len, small_piece; /* step 2: q and the small-piece length */
  int32_t warps_per_cta;        /* decode warps per CTA (step 5) */
  int32_t prefill_parts_target; /* split-K target parts per q tile (step 1; 1 = no split) */
  int64_t num_units;
  double sim_seconds;   /* T_sim (step 6) */
  double seconds;       /* t_hat */
} niyama_predict_info;
niyama_status niyama_predict_detail(const niyama_predictor* p, const niyama_batch_desc* desc, niyama_predict_info* out);
/* Full iteration (§8(f) rank 4; the paper's predictor covers the whole iteration, P:319,
 * P:672): with layers > 0, niyama_predict_iter_time (and everything built on it: the
 * chunk choice, the scheduler) returns
 *     t_iter = c0 + c1 * T + lin(T) + layers * t_hat(batch)
 * where T = rows of the batch, t_hat the attention model above, and lin the MEASURED time of
 * one iteration's linear layers at T tokens (a profile lookup table: n >= 2 points
 * (tokens ascending, > 0), piecewise linear, extrapolated linearly beyond the ends).
 * layers = 0 restores the single attention launch.  EINVAL on a malformed table. */
niyama_status niyama_predictor_set_iteration(niyama_predictor* p, int32_t layers, const int32_t* tokens,
                                             const double* seconds, int32_t n, double c0, double c1);
/* (c0, c1) by least squares on relative residuals of measured full iterations (host arrays;
 * the table and layers must be set first); writes them into the predictor. */
niyama_status niyama_predictor_fit_iteration(niyama_predictor* p, const niyama_batch_desc* batches,
                                             const double* seconds, int32_t n);
/* a1 — chunk for the batch {C prefill rows at chunk_offset} + desc's decodes
 * (desc's prefill slices are ignored) against slack_s (a latency equal to the
 * slack is feasible, R18; 1e-12 relative guard).  cap = max(0, min(max_chunk,
 * prefill_remaining)).  If C = 0 is infeasible: chunk_out = 0, infeasible_out
 * = 1 (a flag, not an error).  Else if cap is feasible: cap.  Else
 * bisection lo = 0, hi = cap, mid = floor((lo+hi)/2) until hi = lo + 1:
 * returns lo, so t_hat(C) <= slack < t_hat(C+1) (S:137 inverse consistency);
 * C is the largest feasible chunk whenever t_hat is non-decreasing in C. */
niyama_status niyama_max_feasible_chunk(const niyama_predictor* p, const niyama_batch_desc* decodes_only,
                                        int32_t chunk_offset, int32_t prefill_remaining, double slack_s,
                                        int32_t max_chunk, int32_t* chunk_out, int32_t* infeasible_out);
void niyama_predictor_destroy(niyama_predictor* p);
/* Model the launches of this kv: its device's SM count (default NIYAMA_PRED_SMS) and
 * its current niyama_tuning (default tuning otherwise).  EINVAL if the predictor's
 * local shape (Hq/G, Hkv/G, head_dim, dtype) differs from the kv's. */
niyama_status niyama_predictor_bind(niyama_predictor* p, const niyama_kv* kv);

/* a1 — slack of the running decodes (§3.3; Eq. 1-3).
 * Interactive decode: D_n - now with D_n = t_arrival + TTFT + (n-1)*TBT (Eq. 2)
 * and n = next_token.  Non-interactive: (D_total - now)/max(1, est_remaining)
 * with D_total = t_arrival + TTLT (Eq. 3; pacing bound R17).  Result: the
 * minimum over decodes, +INFINITY for n = 0. */
typedef struct {
  int32_t interactive;   /* 1 = TTFT/TBT class, 0 = TTLT class */
  int32_t next_token;    /* 1-based token position n produced by this iteration */
  int32_t est_remaining; /* non-interactive: estimated tokens still to decode */
  int32_t reserved;
  double t_arrival, slo_ttft, slo_tbt, slo_ttlt; /* seconds */
} niyama_decode_qos;
niyama_status niyama_min_slack(const niyama_decode_qos* decodes, int32_t n, double now, double* slack_out);


/* ===================================================================== §8(f)1
 * QoS scheduler core (per replica; P:205 pipeline ①-⑦).  Each iteration:
 * ① order the prefill queue by the policy's key (NIYAMA: hybrid priority Eq. 4
 * P:264 interactive P = t_arrival + TTFT + alpha*Prefill_rem, Eq. 5
 * non-interactive P = t_arrival + TTLT + alpha*(Prefill_rem + Decode_rem), the
 * decode estimate being mean + 2 std of the app's completed decode lengths,
 * P:276; FCFS / EDF / SJF / SRPF baselines; ties by arrival
 * then id); ② check violations (Violated: deadline < now; WillViolate:
 * deadline < now + Prefill_rem + decode_token_s (TTFT; + Decode_rem instead for
 * TTLT), R23); ③ eager
 * relegation (Low-priority violators first, High ones only in an
 * iteration that relegated no Low one, R22); the relegated queue is served
 * (earliest original deadline first) only when no primary candidate is left
 * (R28); selective preemption (R26); ④ dynamic chunking: the largest
 * chunk whose predicted batch latency fits the min slack of the running
 * decodes (bisection as niyama_max_feasible_chunk; relegated decodes do
 * not bind, R29; an interactive decode already past its token deadline binds at
 * its TBT, R31), or fixed_chunk; ⑤ greedy multi-fill (R27; the last
 * slice is shrunk if the filled batch predicts above the slack); ⑦ complete():
 * each running decode emitted one token; finished ones leave (their length
 * feeds the history); completed prefills enter the decode queue (R21).
 * Prefill_rem = the cost model's prefill-only time of the remaining prompt in
 * max_chunk pieces (R24); Decode_rem = estimated tokens x decode_token_s (R25).
 * Request ids are the KV cache's sequence ids.  Single-threaded. */
typedef enum {
  NIYAMA_POLICY_NIYAMA = 0, NIYAMA_POLICY_FCFS = 1, NIYAMA_POLICY_EDF = 2, NIYAMA_POLICY_SJF = 3,
  NIYAMA_POLICY_SRPF = 4
} niyama_policy;
typedef enum { NIYAMA_PREEMPT_NEVER = 0, NIYAMA_PREEMPT_SELECTIVE = 1, NIYAMA_PREEMPT_ALWAYS = 2 } niyama_preemption;
typedef enum { NIYAMA_QOS_OK = 0, NIYAMA_VIOLATED = 1, NIYAMA_WILL_VIOLATE = 2 } niyama_qos_status;
typedef struct {
  int32_t policy;               /* niyama_policy */
  int32_t preemption;           /* niyama_preemption (ALWAYS = priority order alone) */
  int32_t dynamic_chunk;        /* 1 = slack-driven chunk; 0 = fixed_chunk (Sarathi baselines) */
  int32_t fixed_chunk;          /* tokens, >= 0 */
  int32_t max_chunk;            /* tokens, >= 1 (2K) */
  int32_t relegation;           /* eager relegation on/off */
  int32_t multi_fill;           /* several prefill slices per batch */
  int32_t history_min_samples;  /* completions per app before the history replaces the prior */
  double alpha;                 /* Eq. 4-5 weight, >= 0 (s of deadline per s of remaining work) */
  double prior_mean, prior_std; /* decode-length prior (tokens) */
  double decode_token_s;        /* seconds per decode iteration in Decode_rem (R25) */
  double layers;                /* an iteration = fixed_s + layers x the predictor's batch time (R30), > 0 */
  double fixed_s;               /* >= 0 */
  int64_t kv_token_budget;      /* KV admission (R32): 0 = unlimited; else prefill slices are cut so that the
                                   tokens held by unfinished requests plus the batch's new tokens stay <= this */
} niyama_sched_config;
typedef struct {
  int32_t interactive;          /* 1: TTFT + TBT (Eq. 1-2); 0: TTLT (Eq. 3) */
  int32_t reserved;
  double slo_ttft, slo_tbt, slo_ttlt; /* seconds */
} niyama_qos_spec;
typedef struct niyama_sched niyama_sched;
typedef struct {
  niyama_batch_desc desc;       /* ready for niyama_plan_create; arrays owned by the scheduler, valid until the
                                   next next_batch / destroy.  Slices in fill order, decodes by (arrival, id);
                                   tier = the request's submit tier. */
  int32_t chunk_budget;         /* ④ budget (before the fill) */
  int32_t infeasible;           /* 1: even a decode-only batch predicts above the slack (budget 0) */
  double predicted_s;           /* the cost model on desc */
  double min_slack_s;           /* +INF without binding decodes */
  int32_t num_relegated;        /* ids relegated by this call */
  const int64_t* relegated;
} niyama_sched_batch;
typedef struct {
  int32_t state;                /* 0 prefill queue, 1 decode queue, 2 relegated queue, 3 done */
  int32_t relegated, prefill_done, decoded, prompt, low;
} niyama_request_info;

void niyama_sched_config_default(niyama_sched_config* cfg); /* NIYAMA, selective, dynamic, 256/2048, relegation,
                                                               multi-fill, 30, alpha 0, prior 415 +- 300, 50 ms,
                                                               layers 1, fixed 0 */
/* model: borrowed (must outlive the scheduler).  EINVAL on a bad config. */
niyama_status niyama_sched_create(const niyama_sched_config* cfg, const niyama_predictor* model, niyama_sched** out);
void niyama_sched_destroy(niyama_sched* s);
/* ① a request arrives (prompt >= 1, new id).  tier 0..255 is copied to the batch desc. */
niyama_status niyama_sched_submit(niyama_sched* s, int64_t id, double t_arrival, int32_t prompt_tokens,
                                  const niyama_qos_spec* qos, int32_t low_priority, int32_t app_id, int32_t tier);
/* ①-⑤ build the iteration's batch at time `now` (ESTATE if the previous non-empty batch was not completed).
 * An empty batch (no slices, no decodes) needs no complete(). */
niyama_status niyama_sched_next_batch(niyama_sched* s, double now, niyama_sched_batch* out);
/* ⑦ the outstanding batch ran and ended at `now`; finished = its decodes that emitted their last token
 * (EINVAL for any other id; validated before any change). */
niyama_status niyama_sched_complete(niyama_sched* s, double now, const int64_t* finished, int32_t n_finished);
niyama_status niyama_sched_request(const niyama_sched* s, int64_t id, niyama_request_info* out);
niyama_status niyama_sched_counts(const niyama_sched* s, int32_t* counts4); /* requests per state */
/* The request's policy key at its current state and its violation status at `now` (tests, tools). */
niyama_status niyama_sched_priority(niyama_sched* s, int64_t id, double now, double* key_out, int32_t* status_out);

#ifdef __cplusplus
}
#endif
#endif /* NIYAMA_H_ */
