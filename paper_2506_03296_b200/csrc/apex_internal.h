// Internal interface between the host core (apex_host.cpp) and the CUDA
// launchers (append.cu, decode.cu, synth.cu).  Not part of the ABI.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/apex.h"

namespace apex {

constexpr int kBlock = 16;          // tokens per KV block (reading c9)
constexpr int kHeadDim = 128;       // D
constexpr int kMaxLayers = 64;
constexpr int kMaxOut = 8;          // destinations of apex_decode_attention_ex

// One split-KV work item: the tokens of logical blocks [blk0, blk0+nblk) of
// (batch row b, kv head g).  32 bytes, read once per item by the decode kernel.
struct __align__(16) WorkItem {
    int32_t b;        // batch row (q/out row)
    int32_t g;        // kv head
    int32_t blk0;     // first logical block
    int32_t nblk;     // blocks in this item (>= 1)
    int32_t part;     // partial slot, or -1 if the item covers the whole (b, g) pair
    int32_t seq;      // sequence id (block_table row)
    int32_t len;      // tokens of the sequence (masking of the last block)
    int32_t mg;       // index into the merge list (split items), or -1
};

// A work item as uploaded: the item plus the physical ids of its first kInlineIds
// blocks (-1 past nblk), so the producer can issue the first TMA loads in the same
// round trip as the item instead of after a dependent block-table load.
constexpr int kInlineIds = 8;
struct __align__(16) ItemRec {
    WorkItem it;
    int32_t ids[kInlineIds];
};

// One (b, g) pair whose items were split: partial slots [part0, part0+nparts).
// The last item of the pair to finish merges the partials inside the decode kernel.
struct __align__(16) MergeItem {
    int32_t b, g, part0, nparts;
};

// Per-step counts, uploaded with the work list.  Kernels read them from device
// memory so every launch of apex_kv_append / apex_decode_attention has
// step-invariant parameters (fixed pointers, fixed grids): a captured CUDA graph
// of the per-layer launches stays valid across steps; only apex_kv_alloc (host
// planning + H2D upload) runs outside the graph.
struct __align__(16) StepHeader {
    int32_t n_items;
    int32_t n_merges;
    int32_t n_rows;       // new-token rows of the step (append)
    int32_t o_merges;     // byte offsets from the header of this step's merge list and slot map:
    int32_t o_slots;      // the upload is packed (ONE H2D copy per step); kernels derive the
    int32_t pad[3];       // pointers on the device, so their launch parameters stay fixed
};
// Right after the header (at byte kCtaBeginOffset of the upload region): int32
// cta_begin[grid + 1].  CTA c first runs items [cta_begin[c], cta_begin[c+1])
// (its static range), then pulls items cta_begin[grid] + atomicAdd(queue) until
// the list ends.
constexpr int kCtaBeginOffset = 32;

struct DecodeParams {
    const void *q;             // [B][Hq][D]
    void *out[8];              // n_out destinations (local and/or peer-mapped), each written identically
    int64_t out_row_stride;    // elements between consecutive batch rows of a destination
    int64_t out_head_stride;   // elements between consecutive heads (D: row-major [B][H][D]; B*D: head-major)
    int32_t out_head_offset;   // head index of this handle's q-head 0 inside a destination
    int32_t n_out;
    // completion signal (f3): when signals[0] != nullptr, after every output row of the
    // call is stored in every destination, signals[i][signal_slot] = signal_value
    // (system-scope release) for i < n_out; sig_counter counts finished CTAs (left at 0)
    uint32_t *signals[8];
    int32_t signal_slot;
    uint32_t signal_value;
    int32_t *sig_counter;
    const int32_t *block_table;
    const ItemRec *items;
    const MergeItem *merges;   // unused (the kernels derive the list from hdr->o_merges)
    float *part_o;             // [slots][G][D]   unnormalised sum_t p_t v_t (fp32)
    float *part_ml;            // [slots][G][2]   (running max m in log2 units, sum l)
    int32_t *counters;         // [2]: work-queue head, CTAs done
    int32_t *merge_counters;   // [n_merges]: split items finished per pair (left at 0)
    const StepHeader *hdr;     // this step's counts (device, written by apex_kv_alloc's upload)
    const int32_t *cta_begin;  // [grid + 1] static item ranges, then the dynamic queue base
    int32_t merge_grid;        // fixed grid of the merge kernel (grid-stride over hdr->n_merges)
    int32_t max_blocks_per_seq;
    int32_t num_q_heads;
    int32_t num_kv_heads;
    float scale_log2;          // scale * log2(e)
    int32_t tma_segs;          // 1: one 3-D TMA op per tile; n: n 2-D ops (one per 128-B segment)
    int32_t fuse_merge;        // 1: last split per pair merges in-kernel; 0: apex_merge_kernel launch
    // fused append (apex_decode_attention_append; every sequence of the step has
    // exactly one new token, row b of k_new/v_new [B][Hkv][D]): the CTA that loads a
    // sequence's last block writes the new K/V row into the pool (producer) and
    // patches it into the shared-memory tile (consumer) before using it
    const void *k_new;         // nullptr: no fused append
    const void *v_new;
    void *kv_pool;             // this layer's pool
    int32_t num_blocks;
};

struct TmaMap {
    CUtensorMap kv;            // 64-byte aligned opaque descriptor of one layer's KV pool
};

// sets the thread-local apex_last_error() text and returns st
apex_status set_error(apex_status st, const char *fmt, ...);

// launchers: return cudaSuccess or the launch error
cudaError_t launch_upload(const void *host_src, void *dev_dst, size_t bytes, const int2 *bt_delta, int n_bt,
                          const int2 *len_delta, int n_len, int32_t *block_table, int32_t *seq_lens, int sm_count,
                          cudaStream_t s);
cudaError_t launch_apply_deltas(const int2 *bt_delta, int n_bt, const int2 *len_delta, int n_len,
                                int32_t *block_table, int32_t *seq_lens, cudaStream_t s);
cudaError_t launch_append(apex_dtype dt, const void *k_new, const void *v_new, void *kv_pool,
                          const int32_t *slots, const StepHeader *hdr, int n_kv_heads, int sm_count,
                          cudaStream_t s);
cudaError_t launch_decode(apex_dtype dt, int group, const TmaMap &tm, const DecodeParams &p,
                          int grid, cudaStream_t s);
// completion signals (signal.cu): wait until every signals[i] >= value (i < n), or post
// value into slot `slot` of each of the n_dst arrays; `status` (device, may be null)
// receives 1 if the wait gave up after timeout_ns
cudaError_t launch_signal_wait(const uint32_t *signals, int n, uint32_t value, uint64_t timeout_ns,
                               uint32_t *status, cudaStream_t s);
cudaError_t launch_signal_post(uint32_t *const *dst, int n_dst, int slot, uint32_t value, cudaStream_t s);
// persistent-grid size the decode kernel of (dtype, group) runs with on this device
int decode_grid_ctas(apex_dtype dt, int group, int sm_count);
bool decode_supported(apex_dtype dt, int group);
// attribute setup + eager loading of every kernel a handle may launch (CUDA lazy
// loading would load a kernel at its first launch, which can block behind a spinning
// apex_signal_wait kernel and deadlock until its timeout)
cudaError_t decode_prepare(apex_dtype dt, int group);
cudaError_t append_prepare();
cudaError_t signal_prepare();

}  // namespace apex
