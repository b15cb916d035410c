/*
 * apex.h — C ABI of the B200-native APEX decode-attention hot path.
 *
 * What the library computes (PAPER.md = /root/reference/PAPER.md, "P:n" = line n):
 *   Decode-phase self-attention over a growing KV cache (§2.1: each
 *   layer caches one K and one V vector per token; decode generates one token
 *   per step), memory-bandwidth-bound (§2.2), with GQA K/V sharing,
 *   the cache managed in fixed-size blocks like the paper's "Paged Attention"
 *   backends (§4.1) and handled dynamically (§3.1), plus the
 *   profiling-informed time prediction of §3.1/§3.2.
 *   Per request b and query head h (kv head g = h / (Hq/Hkv)):
 *       out[b,h,:] = softmax_t(scale * q[b,h,:] . K[b,g,t,:]) . V[b,g,t,:]
 *   over t = 0 .. len_b-1 (BASELINE.json north_star states the formula;
 *   DESIGN.md "Readings" c1-c16 list every interpretation of a silence).
 *
 * Conventions
 *   - Every call returns apex_status; nothing throws or aborts across the ABI.
 *     On a non-OK status apex_last_error() returns a thread-local message.
 *   - Device pointers are CUDA device addresses owned by the CALLER (here:
 *     torch tensors).  Host pointers are plain host memory, read during the
 *     call only.  `stream` is a cudaStream_t passed as void* (NULL = legacy
 *     default stream); every device operation is enqueued on it and no call
 *     synchronises the device.
 *   - All calls that enqueue work for one handle must be issued on one stream
 *     (or ordered by the caller): apex_kv_alloc uploads the step's metadata into
 *     the workspace that apex_kv_append / apex_decode_attention read.
 *   - A handle is not thread-safe; use one handle per (process, GPU, model).
 *   - CUDA graphs: every launch made by apex_kv_append / apex_decode_attention
 *     has step-invariant parameters (the step's counts are read from a device
 *     header that apex_kv_alloc uploads; grids and workspace offsets are fixed),
 *     so the per-layer calls may be captured once and replayed every step with
 *     apex_kv_alloc called outside the graph before each replay.  q/out/k_new/
 *     v_new must then be the same (static) buffers at every replay.
 *   - Host-only handles (desc.kv_pool == NULL and desc.block_table == NULL) run
 *     the allocator and planner without any CUDA call; append/decode then
 *     return APEX_EINVAL.  Used by CPU tests and host-side planning.
 */
#ifndef APEX_H
#define APEX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    APEX_OK = 0,
    APEX_EINVAL = 1,        /* bad argument / state; nothing was changed or enqueued */
    APEX_ENOBLOCKS = 2,     /* KV pool exhausted; the alloc call changed nothing */
    APEX_ESEQ = 3,          /* unknown or already-released sequence id */
    APEX_ECUDA = 4,         /* a CUDA runtime/driver call or launch failed */
    APEX_EUNSUPPORTED = 5   /* valid but unsupported shape/dtype combination */
} apex_status;

typedef enum { APEX_F32 = 0, APEX_F16 = 1, APEX_BF16 = 2 } apex_dtype;  /* KV, q and out share it */

typedef struct apex_kv apex_kv;
typedef struct apex_cost apex_cost;
typedef void *apex_stream;   /* cudaStream_t */

typedef struct {
    int32_t num_layers;          /* physical layers that own a KV pool (1..64) */
    int32_t num_q_heads;         /* Hq (local to this rank when heads are sharded) */
    int32_t num_kv_heads;        /* Hkv; Hq % Hkv == 0, group g = Hq/Hkv in {1,2,4,8} */
    int32_t head_dim;            /* D; must be 128 */
    int32_t block_size;          /* tokens per KV block; must be 16 (reading c9) */
    int32_t num_blocks;          /* blocks in each pool */
    int32_t max_seqs;            /* sequence ids are 0 .. max_seqs-1 (rows of block_table) */
    int32_t max_blocks_per_seq;  /* columns of block_table; max context = this * block_size */
    int32_t max_batch;           /* max sequences in one apex_kv_alloc call (decode batch) */
    int32_t max_new_tokens;      /* max sum(n_new) in one apex_kv_alloc call */
    apex_dtype dtype;
    /* [num_layers] device pointers, one KV pool per physical layer, each
       [num_blocks][Hkv][2][block_size][D] elements of `dtype` (index 0 = K,
       1 = V), 128-byte aligned: the K and V rows of one (block, kv head) are
       one contiguous 2*16*D-element tile, fetched by a single TMA.  Pools may
       alias (logical layers mapped onto fewer physical layers is the caller's
       choice). */
    void *const *kv_pool;
    int32_t *block_table;        /* device int32 [max_seqs][max_blocks_per_seq] */
    int32_t *seq_lens;           /* device int32 [max_seqs] */
    void *workspace;             /* device scratch, >= apex_kv_workspace_bytes(desc), 256-B aligned */
    size_t workspace_bytes;
} apex_kv_desc;

/* Device workspace the handle needs for this desc (step metadata, work list,
   split-KV partials).  Returns 0 if the desc is invalid. */
size_t apex_kv_workspace_bytes(const apex_kv_desc *desc);

/* Validate the desc, build the LIFO free list (first pop = block 0, reading
   c10), the host mirrors, the pinned staging ring and one TMA descriptor per
   physical layer; load every kernel the handle may launch (so no later launch
   waits on CUDA lazy module loading, e.g. behind a spinning apex_signal_wait);
   zero the workspace's queue / merge / signal counters (cudaMemset, then a
   device synchronise: create is not on the hot path and the counters must be
   zero before any stream uses them).  The pools' contents are not touched
   (callers may pre-fill them, e.g. with NaN in tests). */
apex_status apex_kv_create(const apex_kv_desc *desc, apex_kv **out);

/* Free host state.  The caller must synchronise its streams first. */
void apex_kv_destroy(apex_kv *kv);

/* Reserve slots for this step and DEFINE THE STEP BATCH.
   seq_ids[i] (unique, 0..max_seqs-1) gains n_new[i] >= 0 tokens; a sequence
   with length 0 is new.  Batch row i of q/out is seq_ids[i]; the k_new/v_new
   rows of apex_kv_append are the n_new[i] rows of each seq, concatenated in
   call order.  A block is popped only when a token lands at pos % 16 == 0.
   All-or-nothing: APEX_ENOBLOCKS / APEX_EINVAL leave every state unchanged.
   Lengths after the call must be in [1, max_blocks_per_seq*16].  Enqueues ONE
   kernel on `stream`: it reads the step metadata (block-table/length deltas,
   slot mapping, split-KV work list) straight from the handle's mapped pinned
   staging buffer (zero-copy), writes it into the workspace and applies the
   deltas to block_table / seq_lens (an H2D copy + a delta kernel before: C1
   step 40 -> 30 us).  The staging buffer is double-buffered; reusing one waits
   (host) for the kernel that read it two calls earlier.  Host work reuses
   scratch storage kept by the handle (no per-step allocations once warm).
   n in [1, max_batch]. */
apex_status apex_kv_alloc(apex_kv *kv, const int32_t *seq_ids, const int32_t *n_new, int32_t n,
                          apex_stream stream);

/* Return the sequence's blocks to the free list in reverse table order (so
   they are popped again in table order) and forget it.  Host-only: the device
   block_table row is left stale (it is never read for a released sequence). */
apex_status apex_kv_release(apex_kv *kv, int32_t seq_id);

/* Write this step's new K and V vectors of physical layer `layer` into the
   pools (one K and one V vector per token per layer).  k_new, v_new:
   device [sum(n_new)][Hkv][D] of dtype, rows ordered as defined by the last
   apex_kv_alloc.  Bit-exact copy: kv_pool[layer][blk][h][0][t][:] = k_new[row][h][:]
   and kv_pool[layer][blk][h][1][t][:] = v_new[row][h][:], with (blk, t) from the
   row's slot.  One kernel launch. */
apex_status apex_kv_append(apex_kv *kv, int32_t layer, const void *k_new, const void *v_new,
                           apex_stream stream);

/* Decode attention of the last alloc's batch against physical layer `layer`.
   q: device [B][Hq][D] of dtype (post-RoPE queries, one row per seq in alloc
   order); out: device [B][Hq][D] of dtype (rounded to nearest even once, from
   fp32).  Attends over seq_lens[seq] tokens, INCLUDING this step's appended
   token (reading c3).  scale is usually 1/sqrt(D) (reading c1).  Split-KV
   flash-decode (FlashDecoding lineage): one persistent kernel over the
   planned work items, plus one log-sum-exp merge kernel for the split
   (seq, kv-head) pairs -- or, for small steps (latency regime), the merge is
   done inside the decode kernel by the last split to finish (see
   apex_kv_decode_launches).  Results are deterministic and independent of the physical
   block placement.  Supported: F32 with g == 1 (CUDA cores), F16 with
   g == 1 and F16/BF16 with g in {2,4,8} (tensor cores, mma.sync with the
   q-group on the N side; MHA with one live column); otherwise
   APEX_EUNSUPPORTED.
   CUDA graphs: every launch parameter is step-invariant within a regime, so a
   captured sequence of calls stays valid while apex_kv_decode_launches() is
   unchanged (the regime switches at T = 512 tiles per CTA). */
apex_status apex_decode_attention(apex_kv *kv, int32_t layer, const void *q, void *out,
                                  float scale, apex_stream stream);

/* As apex_decode_attention, but the output D-vector of (batch row b, local q head
   h) is written to each of the n_out (1..8) destinations outs[i] at element offset
       b*out_row_stride + (out_head_offset + h)*out_head_stride
   (row-major [B][H][D]: row stride H*D, head stride D; head-major [H][B][D]: row
   stride D, head stride B*D).  Strides are in elements, multiples of 4, and rows /
   heads must not overlap (out_head_stride >= D and out_row_stride >= (offset+Hq) *
   head stride, or out_row_stride >= D and out_head_stride >= B * row stride);
   destinations 16-byte aligned.  Head sharding: rank r writes
   its head slice head-major into a local [Hq/N][B][D] buffer that NCCL all-gathers
   into [Hq][B][D] with no permute; or (f3) it passes the symmetric, peer-mapped
   [Hq][B][D] buffers of all ranks with out_head_offset = r*Hq/N, so the all-gather
   happens inside the epilogue.
   signals: NULL, or n_out device pointers (peer-mapped allowed) to uint32 arrays;
   after every output row of this call is stored in every destination, the call's
   last launch writes signals[i][signal_slot] = signal_value with a system-scope
   release (one in-kernel completion flag per layer-call, no host barrier).  A
   reader waits with apex_signal_wait before it reads the rows.  Other errors as
   apex_decode_attention; APEX_EINVAL on overlapping strides or bad signals. */
apex_status apex_decode_attention_ex(apex_kv *kv, int32_t layer, const void *q, void *const *outs, int32_t n_out,
                                     int64_t out_row_stride, int64_t out_head_stride, int32_t out_head_offset,
                                     uint32_t *const *signals, int32_t signal_slot, uint32_t signal_value,
                                     float scale, apex_stream stream);

/* Enqueue on `stream` a one-warp kernel that waits until every signals[i] (device
   uint32, i < n) has reached `value` (wrap-safe: (int32_t)(signals[i] - value) >= 0)
   with system-scope acquire loads, so later work on the stream sees the rows the
   signalling launches stored (f3 completion flag; PAPER.md P:82 analogue).  If
   timeout_ns elapses first the kernel stops waiting and, if status != NULL,
   writes 1 to the device word *status (callers check it; nothing hangs).
   APEX_EINVAL on NULL/misaligned pointers or n < 1. */
apex_status apex_signal_wait(const uint32_t *signals, int32_t n, uint32_t value, uint64_t timeout_ns,
                             uint32_t *status, apex_stream stream);

/* Enqueue a kernel that writes `value` into dst[i][slot] (i < n_dst <= 8, device or
   peer-mapped uint32 arrays) with a system-scope release, after everything earlier
   on `stream`.  Used by a reader to hand a consumed symmetric buffer back to the
   writers (write-after-read guard of the fused gather). */
apex_status apex_signal_post(uint32_t *const *dst, int32_t n_dst, int32_t slot, uint32_t value, apex_stream stream);

/* apex_kv_append + apex_decode_attention in ONE launch for
   a pure decode step: every sequence of the last apex_kv_alloc has exactly one
   new token (else APEX_EINVAL, nothing enqueued).  k_new / v_new: device
   [batch][Hkv][D] in the step's row order, 16-byte aligned.  Latency regime
   (apex_kv_decode_launches() == 1): ONE launch -- the CTA that streams a
   sequence's last block writes the new K/V row into the pool (so later steps
   see it, exactly as apex_kv_append would) and patches it into its
   shared-memory copy of the tile before use.  Bandwidth regime: the append
   kernel then the plain decode kernel (measured faster there).  Either way
   outputs and pools are bit-identical to the two-call sequence.  Other
   arguments as apex_decode_attention. */
apex_status apex_decode_attention_append(apex_kv *kv, int32_t layer, const void *q, const void *k_new,
                                         const void *v_new, void *out, float scale, apex_stream stream);

/* ---- planner knobs and introspection (host state only; no CUDA calls) ---- */

/* Split-KV chunk in tokens (multiple of 16) used by the NEXT apex_kv_alloc;
   0 = automatic.  A fixed chunk makes results bit-identical across request /
   head sharding (tests).  APEX_EINVAL if not a multiple of block_size or < 0. */
apex_status apex_kv_set_split(apex_kv *kv, int32_t chunk_tokens);
/* Number of persistent CTAs the planner targets and the decode kernel launches
   with (0 = device default).  Takes effect at the NEXT apex_kv_alloc. */
apex_status apex_kv_set_grid(apex_kv *kv, int32_t ctas);
/* Bandwidth-regime scheduling used by the NEXT apex_kv_alloc (ignored in the
   latency regime and with a forced split chunk):
     dyn_permille = -1: every (row, kv-head) pair cut into ~16 items per CTA,
                        pulled longest-first from a device queue (FlashDecoding-
                        style dynamic split);
     dyn_permille = -2: "guided" (default): as -1 with ~8 items per CTA, except that
                        the pairs holding the last 10% / 5% / 2% of the tiles are
                        cut into 1/2, 1/4, 1/8-size items, so the queue ends with
                        small items;
     dyn_permille in [0, 1000]: "stream-K" -- the first (1000 - dyn_permille)
                        permille of the tiles, in (row, kv-head, block) order,
                        are cut into one contiguous static range per CTA (no
                        queue traffic, ~T/P tiles each); the rest are small items
                        pulled from the queue after a CTA's static range.
   Default: the automatic choice documented in DESIGN.md.  APEX_EINVAL outside
   [-2, 1000]. */
apex_status apex_kv_set_sched(apex_kv *kv, int32_t dyn_permille);
/* Planner constants (tuning; defaults 512, 4, 900, 950, 980), used by the NEXT
   apex_kv_alloc: the latency regime (fused in-kernel merge, one launch) applies
   while total tiles T <= latency_tiles_per_cta * grid (0 disables it); the guided
   bandwidth split cuts items of ceil(T / (guided_div * grid)) blocks, and, for the
   pairs holding the last (1000 - pm1), (1000 - pm2), (1000 - pm3) permille of the
   tiles, items of 1/2, 1/4, 1/8 of ceil(T / (max(guided_div, 8) * grid)) blocks.  APEX_EINVAL (nothing changed) unless
   0 <= latency_tiles_per_cta <= 2^20, 1 <= guided_div <= 64 and
   0 <= pm1 <= pm2 <= pm3 <= 1000. */
apex_status apex_kv_set_planner(apex_kv *kv, int32_t latency_tiles_per_cta, int32_t guided_div, int32_t guided_pm1,
                                int32_t guided_pm2, int32_t guided_pm3);
int32_t apex_kv_num_free_blocks(const apex_kv *kv);
/* len and block ids (table order) of a live sequence; *n_blocks may exceed cap
   (then only cap ids are written). */
apex_status apex_kv_seq_info(const apex_kv *kv, int32_t seq_id, int32_t *len, int32_t *blocks,
                             int32_t cap, int32_t *n_blocks);
/* slot (= block*block_size + offset) of every new-token row of the last alloc */
apex_status apex_kv_last_slots(const apex_kv *kv, int32_t *slots, int32_t cap, int32_t *n);
/* last alloc's work list: 6 int32 per item {batch row, kv head, first logical
   block, n blocks, partial slot or -1, seq id}, in execution-priority order */
apex_status apex_kv_plan(const apex_kv *kv, int32_t *items, int32_t cap, int32_t *n_items,
                         int32_t *n_merges);

/* last alloc's per-CTA static ranges: *n = grid + 1 entries cta_begin[] (CTA c
   runs items [cta_begin[c], cta_begin[c+1]) of apex_kv_plan's list first; items
   from cta_begin[grid] on are pulled from the device queue).  At most cap
   entries are written. */
apex_status apex_kv_plan_ranges(const apex_kv *kv, int32_t *cta_begin, int32_t cap, int32_t *n);

/* Kernel launches the next apex_decode_attention will issue for the last alloc's
   plan: 1 (decode kernel; LSE merge fused in-kernel, latency regime) or 2
   (decode kernel + merge kernel; the merge kernel exits at once if the step has
   no split pairs).  Returns -1 if no step is allocated. */
int32_t apex_kv_decode_launches(const apex_kv *kv);

/* ---- profiling-informed time prediction ---- */

/* Table of measured per-layer-call decode-attention times us[i*nk + j] at
   (batch[i], kv_tokens[j]).  Grids strictly increasing and positive; times
   finite and > 0; nb, nk >= 1.  Copies the table. */
apex_status apex_cost_create(const int32_t *batch, int32_t nb, const int64_t *kv_tokens, int32_t nk,
                             const double *us, apex_cost **out);
/* Bilinear interpolation over (batch, total kv tokens of the batch), clamped to
   the grid's edges on each axis (reading c16).  Pure host computation. */
apex_status apex_predict_time(const apex_cost *cost, int32_t batch, int64_t kv_tokens,
                              double *us_out);
/* Online recalibration from one measured per-layer-call time (§6:
   online profiling to correct the offline profile's mispredictions; the update
   rule is DESIGN.md reading c17):
     1. if (batch, kv_tokens) lies outside the grid on an axis, a grid line through
        it is added on that axis, valued at the current (clamped) predictions --
        no prediction changes;
     2. with e = measured_us - predicted and w_c the bilinear weights of the four
        corners of the point's cell, corner c += alpha * e * w_c / sum_c w_c^2
        (normalised LMS): the prediction at the point becomes exactly
        predicted + alpha * e; predictions whose cell shares no corner with
        it are unchanged.
   alpha in (0, 1] (1: trust the measurement fully; smaller: EWMA-like smoothing),
   measured_us finite and > 0, at most 256 grid points per axis; otherwise
   APEX_EINVAL and the table is unchanged.  Pure host computation. */
apex_status apex_cost_observe(apex_cost *cost, int32_t batch, int64_t kv_tokens, double measured_us,
                              double alpha);
/* Current grid sizes, and a copy of the grid and times (arrays of nb, nk, nb*nk). */
apex_status apex_cost_size(const apex_cost *cost, int32_t *nb, int32_t *nk);
apex_status apex_cost_table(const apex_cost *cost, int32_t *batch, int64_t *kv_tokens, double *us);
void apex_cost_destroy(apex_cost *cost);

/* ---- APEX decision layer (§3.2 Eq1-Eq6, Algorithm 1) ---- */

typedef enum {
    APEX_STRATEGY_GPU_ONLY = 0,        /* Alg. 1: no CPU-decode requests (or ratio gate closed) */
    APEX_STRATEGY_ASYM_PIPELINE = 1,   /* Asymmetric Pipelining (NEO) */
    APEX_STRATEGY_ASYNC_OVERLAP = 2    /* Asynchronous Overlap */
} apex_strategy;

typedef struct {
    int32_t n_prefill;        /* |P_sch| */
    int32_t n_gpu_decode;     /* |D_gpu_sch| */
    int32_t n_cpu_decode;     /* |D_cpu_sch| */
    double n_g, n_c;          /* N_G, N_C: GPU / CPU attention rates, tokens per us */
    double t_glinear;         /* T_glinear, us per layer (decode-only profile) */
    double t_gatt;            /* T_gatt,   us per layer (decode-only profile) */
    double t_glinear_pref;    /* T_glinear_pref (Alg. 1 mixed branch; ignored if n_prefill == 0) */
    double t_gatt_pref;       /* T_gatt_pref */
    double min_cpu_ratio;     /* CPU:GPU request-count gate (8); <= 0 disables the gate */
} apex_sched_input;

typedef struct {
    apex_strategy strategy;
    int32_t gate_closed;      /* 1 if the P:378 ratio gate forced GPU-only */
    double lhs, rhs;          /* the two sides of the inequality evaluated (0 if none) */
    double eq6_threshold;     /* 2 T_l/T_a + 3 + T_a/T_l (decode-only case), else 0 */
} apex_decision;

/* Eq6: AP beats GPU-only in decode-only batches iff N_G/N_C < this. */
apex_status apex_pipelining_threshold(double t_glinear, double t_gatt, double *out);
/* Algorithm 1 exactly as printed: GPU-only if no CPU-decode requests;
   decode-only -> Eq5 decides AP vs AO; mixed -> the modified inequality with
   T_overlap_with_prefill = T_glinear_pref + T_glinear + T_gatt_pref.  Pure host
   function; APEX_EINVAL on non-positive times/rates or negative counts. */
apex_status apex_decide(const apex_sched_input *in, apex_decision *out);

/* Thread-local text for the last non-OK status of this thread ("" if none). */
const char *apex_last_error(void);
const char *apex_version(void);

#ifdef __cplusplus
}
#endif
#endif /* APEX_H */
