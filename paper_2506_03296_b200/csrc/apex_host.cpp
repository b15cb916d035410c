// Host core of the C ABI declared in include/apex.h: paged-KV allocator with a
// host mirror of the block table, split-KV planner, pinned staging of the step
// metadata, TMA descriptor setup, kernel dispatch and the cost model.
//
// Paper anchors (PAPER.md line numbers): KV cache of one K and one V vector per
// token per layer, "handled dynamically" KV management, paged
// attention backends, decode attention, offline
// profiler + performance model.  Allocation contract:
// DESIGN.md reading c10.
#include <algorithm>
#include <cstdlib>
#include <functional>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include <cudaTypedefs.h>

#include "apex_internal.h"

#ifndef APEX_UPLOAD_KERNEL
#define APEX_UPLOAD_KERNEL 1   // 0: cudaMemcpyAsync of the step metadata + the delta kernel
#endif

using apex::MergeItem;
using apex::WorkItem;

namespace {
apex_status vfail(apex_status st, const char *fmt, va_list ap);
}

// thread-local error text for the other translation units (sched.cpp)
apex_status apex::set_error(apex_status st, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vfail(st, fmt, ap);
    va_end(ap);
    return st;
}

namespace {

thread_local std::string g_err;

apex_status vfail(apex_status st, const char *fmt, va_list ap) {
    char buf[512];
    vsnprintf(buf, sizeof buf, fmt, ap);
    g_err = buf;
    return st;
}

apex_status fail(apex_status st, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vfail(st, fmt, ap);
    va_end(ap);
    return st;
}

apex_status cuda_fail(cudaError_t e, const char *what) {
    return fail(APEX_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

int elem_bytes(apex_dtype dt) { return dt == APEX_F32 ? 4 : 2; }

// default bandwidth-regime schedule (apex_kv_set_sched): see DESIGN.md section 7
constexpr int32_t kDefaultDynPermille = -2;

bool desc_host_only(const apex_kv_desc *d) { return d->kv_pool == nullptr && d->block_table == nullptr; }

int query_sm_count(bool host_only) {
    if (host_only) return 148;
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
        cudaGetLastError();
        return 148;
    }
    return n;
}

// Device workspace layout.  Every step uploads one packed region (items,
// merges, slots, block-table deltas, length deltas) into `upload`.
struct WsLayout {
    int32_t max_items = 0, max_merges = 0, max_bt_delta = 0;
    size_t counters = 0, merge_counters = 0, upload = 0, upload_cap = 0, part_o = 0, part_ml = 0, total = 0;
    size_t o_items = 0, o_merges = 0, o_tail = 0;             // offsets inside the upload region
};

WsLayout layout_for(const apex_kv_desc *d, int sm_count) {
    WsLayout w;
    const int G = d->num_q_heads / d->num_kv_heads;
    const int64_t pairs = (int64_t)d->max_batch * d->num_kv_heads;
    // auto planner: items <= pairs + 64 * grid (small pieces) ; grid <= 4 * SMs
    // (stream-K: <= pairs + grid static cuts + pairs + 8 * grid dynamic pieces)
    w.max_items = (int32_t)std::min<int64_t>(2 * pairs + 64LL * 4 * sm_count + 64, 1 << 24);
    w.max_merges = (int32_t)pairs;
    w.max_bt_delta = (int32_t)(cdiv(d->max_new_tokens, d->block_size) + d->max_batch);
    // upload region, fixed offsets: [StepHeader | work items | merges | tail: slots,
    // block-table deltas, length deltas (packed)]; the kernels' pointers into it never move
    // header | cta_begin[grid + 1] (grid <= 4 * SMs) | items ...
    w.o_items = align_up(apex::kCtaBeginOffset + sizeof(int32_t) * (4 * (size_t)sm_count + 1), 256);
    w.o_merges = w.o_items + align_up(sizeof(apex::ItemRec) * (size_t)w.max_items, 256);
    w.o_tail = w.o_merges + align_up(sizeof(MergeItem) * (size_t)w.max_merges, 256);
    size_t up = w.o_tail;
    up += align_up(sizeof(int32_t) * (size_t)d->max_new_tokens, 256);
    up += align_up(sizeof(int2) * (size_t)w.max_bt_delta, 256);
    up += align_up(sizeof(int2) * (size_t)d->max_batch, 256);
    w.counters = 0;                                           // 3 counters x 64 layers (queue, done, signal)
    w.merge_counters = 1024;                                  // one per split pair
    w.upload = align_up(w.merge_counters + sizeof(int32_t) * (size_t)w.max_merges, 256);
    w.upload_cap = up;
    w.part_o = align_up(w.upload + up, 256);
    w.part_ml = align_up(w.part_o + sizeof(float) * (size_t)w.max_items * G * d->head_dim, 256);
    w.total = align_up(w.part_ml + sizeof(float) * 2 * (size_t)w.max_items * G, 256);
    return w;
}

apex_status validate_desc(const apex_kv_desc *d, bool need_workspace = true) {
    if (!d) return fail(APEX_EINVAL, "desc is NULL");
    if (d->num_layers < 1 || d->num_layers > apex::kMaxLayers)
        return fail(APEX_EINVAL, "num_layers %d not in [1, %d]", d->num_layers, apex::kMaxLayers);
    if (d->num_q_heads < 1 || d->num_kv_heads < 1 || d->num_q_heads % d->num_kv_heads)
        return fail(APEX_EINVAL, "num_q_heads %d must be a positive multiple of num_kv_heads %d",
                    d->num_q_heads, d->num_kv_heads);
    if (d->num_kv_heads > 1024 || d->num_q_heads > 4096) return fail(APEX_EINVAL, "too many heads");
    const int G = d->num_q_heads / d->num_kv_heads;
    if (d->head_dim != apex::kHeadDim) return fail(APEX_EUNSUPPORTED, "head_dim %d (only 128)", d->head_dim);
    if (d->block_size != apex::kBlock) return fail(APEX_EUNSUPPORTED, "block_size %d (only 16)", d->block_size);
    if (d->dtype != APEX_F32 && d->dtype != APEX_F16 && d->dtype != APEX_BF16)
        return fail(APEX_EINVAL, "unknown dtype %d", (int)d->dtype);
    if (!apex::decode_supported(d->dtype, G))
        return fail(APEX_EUNSUPPORTED, "dtype %d with group %d (supported: F32/F16 g=1, F16/BF16 g in {2,4,8})",
                    (int)d->dtype, G);
    if (d->num_blocks < 1 || d->max_seqs < 1 || d->max_blocks_per_seq < 1 || d->max_batch < 1 ||
        d->max_new_tokens < 1)
        return fail(APEX_EINVAL, "num_blocks/max_seqs/max_blocks_per_seq/max_batch/max_new_tokens must be >= 1");
    if ((int64_t)d->max_blocks_per_seq * d->block_size > (1LL << 30))
        return fail(APEX_EINVAL, "max context too large");
    if ((int64_t)d->num_blocks * d->num_kv_heads * 2 * d->block_size >= (1LL << 31))
        return fail(APEX_EUNSUPPORTED, "pool rows exceed the TMA coordinate range");
    if (d->max_batch > d->max_seqs) return fail(APEX_EINVAL, "max_batch > max_seqs");
    if (!desc_host_only(d)) {
        if (!d->kv_pool || !d->block_table || !d->seq_lens || (need_workspace && !d->workspace))
            return fail(APEX_EINVAL, "device desc needs kv_pool, block_table, seq_lens, workspace");
        for (int l = 0; l < d->num_layers; ++l) {
            if (!d->kv_pool[l]) return fail(APEX_EINVAL, "pool pointer of layer %d is NULL", l);
            if ((uintptr_t)d->kv_pool[l] & 127)
                return fail(APEX_EINVAL, "pools of layer %d are not 128-byte aligned", l);
        }
        if (need_workspace && ((uintptr_t)d->workspace & 255)) return fail(APEX_EINVAL, "workspace not 256-byte aligned");
    }
    return APEX_OK;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        else
            cudaGetLastError();
    }
    return fn;
}

// TMA view of one pool: rows = ((block*Hkv + head)*2 + {K,V})*16 + t, each row D
// elements.  Preferred 3-D view {128-B segment elements, rows, segments} with
// 128-B swizzle loads a whole (block, head) K+V tile (32 rows) with ONE
// cp.async.bulk.tensor into smem laid out [segment][32 rows][128 B] (K rows
// 0-15, V rows 16-31); the 2-D fallback issues one op per segment into the same
// layout.
bool encode_pool(PFN_cuTensorMapEncodeTiled_v12000 enc, CUtensorMap *m, void *base, apex_dtype dt,
                 int64_t rows, int segs_mode) {
    const int es = elem_bytes(dt);
    const CUtensorMapDataType tdt = dt == APEX_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                    : dt == APEX_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                     : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    const cuuint64_t row_bytes = (cuuint64_t)apex::kHeadDim * es;
    const cuuint32_t seg_elems = 128 / es, segs = (cuuint32_t)(row_bytes / 128);
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r;
    if (segs_mode == 1) {
        cuuint64_t dims[3] = {seg_elems, (cuuint64_t)rows, segs};
        cuuint64_t strides[2] = {row_bytes, 128};
        cuuint32_t box[3] = {seg_elems, (cuuint32_t)(2 * apex::kBlock), segs};   // K and V rows of a tile
        r = enc(m, tdt, 3, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        cuuint64_t dims[2] = {(cuuint64_t)apex::kHeadDim, (cuuint64_t)rows};
        cuuint64_t strides[1] = {row_bytes};
        cuuint32_t box[2] = {seg_elems, (cuuint32_t)(2 * apex::kBlock)};
        r = enc(m, tdt, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    return r == CUDA_SUCCESS;
}

}  // namespace

struct apex_kv {
    apex_kv_desc d{};
    std::vector<void *> kv_pools;
    bool host_only = true;
    int sm_count = 148;
    int group = 1;
    WsLayout ws;
    int32_t forced_chunk_blocks = 0;
    int32_t grid_override = 0;
    int32_t dyn_permille = kDefaultDynPermille;   // apex_kv_set_sched
    int64_t latency_tiles_per_cta = 512;          // latency regime while T <= this * P
    // guided: T/(g0 P) bulk chunk; from permille g1, g2, g3 the halves, quarters, eighths of
    // T/(max(g0, 8) P).  g0 = 4 (was 8, same tail): C2 -0.95%, C3 -0.9%, C4/C5 +-0.05% per
    // call, same box (profiles/r02_guided_div/)
    int32_t guided[4] = {4, 900, 950, 980};
    int32_t plan_grid = 0;                        // CTAs the last plan was made for (= launch grid)
    std::vector<int32_t> cta_begin;               // [plan_grid + 1]

    struct Seq {
        bool live = false;
        int32_t len = 0;
        std::vector<int32_t> blocks;
    };
    std::vector<int32_t> free_stack;   // back() is popped first
    std::vector<Seq> seqs;

    // the current step (defined by the last successful apex_kv_alloc)
    bool have_step = false;
    bool single_token_step = false;   // every sequence of the step has n_new == 1 (fused append allowed)
    int32_t batch = 0, n_rows = 0;
    std::vector<int32_t> batch_seq, slots;
    std::vector<WorkItem> items;
    std::vector<MergeItem> merges;

    // pinned staging ring for the per-step upload
    uint8_t *staging[2] = {nullptr, nullptr};
    uint8_t *staging_dev[2] = {nullptr, nullptr};   // device view of the mapped staging buffers
    cudaEvent_t staged[2] = {nullptr, nullptr};
    bool staged_pending[2] = {false, false};
    int ring = 0;

    // per-step scratch, reused across calls so a step allocates nothing once warm
    // (large std::vectors freed and re-grown every step went back to mmap and page
    // faults: ~2 ms of host time per C5 alloc).  Never observable state: the
    // all-or-nothing contract concerns the fields above.
    struct Scratch {
        std::vector<int32_t> seen, lens, seq_of_row, nblks, pc, cnt, slots, popped;
        std::vector<int2> bt_delta, len_delta;
        std::vector<WorkItem> dyn, items, plan_items;   // queue, sort scratch, spare plan storage
        std::vector<MergeItem> merges;                   // spare plan storage
        std::vector<int32_t> cta_begin;                  // spare plan storage
        std::vector<Seq> before;
        int32_t stamp = 0;
    };
    mutable Scratch sc;

    std::vector<apex::TmaMap> tmaps;
    int tma_segs = 1;   // 1: 3-D map (one op per tile); else ops per tile with the 2-D map
    bool fuse_merge = false;
};

extern "C" {

const char *apex_last_error(void) { return g_err.c_str(); }
const char *apex_version(void) { return "apex-b200 0.1 (sm_100a)"; }

size_t apex_kv_workspace_bytes(const apex_kv_desc *desc) {
    if (validate_desc(desc, false) != APEX_OK) return 0;
    return layout_for(desc, query_sm_count(desc_host_only(desc))).total;
}

apex_status apex_kv_create(const apex_kv_desc *desc, apex_kv **out) {
    if (!out) return fail(APEX_EINVAL, "out is NULL");
    *out = nullptr;
    apex_status st = validate_desc(desc);
    if (st != APEX_OK) return st;
    apex_kv *kv = new (std::nothrow) apex_kv();
    if (!kv) return fail(APEX_EINVAL, "out of host memory");
    kv->d = *desc;
    kv->host_only = desc_host_only(desc);
    kv->group = desc->num_q_heads / desc->num_kv_heads;
    kv->sm_count = query_sm_count(kv->host_only);
    kv->ws = layout_for(desc, kv->sm_count);
    kv->seqs.resize(desc->max_seqs);
    kv->free_stack.resize(desc->num_blocks);
    for (int32_t i = 0; i < desc->num_blocks; ++i) kv->free_stack[i] = desc->num_blocks - 1 - i;
    if (!kv->host_only) {
        if (desc->workspace_bytes < kv->ws.total) {
            delete kv;
            return fail(APEX_EINVAL, "workspace_bytes %zu < required %zu", desc->workspace_bytes,
                        (size_t)apex_kv_workspace_bytes(desc));
        }
        kv->kv_pools.assign(desc->kv_pool, desc->kv_pool + desc->num_layers);
        kv->d.kv_pool = kv->kv_pools.data();
        for (int i = 0; i < 2; ++i) {
            // mapped: the upload kernel reads the step metadata straight from it (zero-copy)
            cudaError_t e = cudaHostAlloc((void **)&kv->staging[i], kv->ws.upload_cap, cudaHostAllocMapped);
            if (e == cudaSuccess) e = cudaHostGetDevicePointer((void **)&kv->staging_dev[i], kv->staging[i], 0);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&kv->staged[i], cudaEventDisableTiming);
            if (e != cudaSuccess) {
                apex_kv_destroy(kv);
                return cuda_fail(e, "apex_kv_create: pinned staging");
            }
        }
        auto enc = get_encode();
        if (!enc) {
            apex_kv_destroy(kv);
            return fail(APEX_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");
        }
        // pool rows: ((block * Hkv + head) * 2 + {K, V}) * 16 + t
        const int64_t rows = (int64_t)desc->num_blocks * desc->num_kv_heads * 2 * desc->block_size;
        kv->tmaps.resize(desc->num_layers);
        for (int mode : {1, 2}) {
            bool ok = true;
            for (int l = 0; l < desc->num_layers && ok; ++l)
                ok = encode_pool(enc, &kv->tmaps[l].kv, kv->kv_pools[l], desc->dtype, rows, mode);
            if (ok) {
                kv->tma_segs = mode == 1 ? 1 : apex::kHeadDim * elem_bytes(desc->dtype) / 128;
                break;
            }
            if (mode == 2) {
                apex_kv_destroy(kv);
                return fail(APEX_ECUDA, "cuTensorMapEncodeTiled rejected the pool layout");
            }
        }
        cudaError_t e = apex::decode_prepare(desc->dtype, kv->group);
        if (e == cudaSuccess) e = apex::append_prepare();
        if (e == cudaSuccess) e = apex::signal_prepare();
        if (e != cudaSuccess) {
            apex_kv_destroy(kv);
            return cuda_fail(e, "apex_kv_create: decode kernel attributes");
        }
        // zero the work-queue and merge counters once; kernels leave them at zero
        e = cudaMemset((uint8_t *)desc->workspace + kv->ws.counters, 0, kv->ws.upload);
        // create is not on the hot path: finish the memset before any launch on any stream
        // (a caller's non-blocking stream is not ordered after the legacy default stream)
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            apex_kv_destroy(kv);
            return cuda_fail(e, "apex_kv_create: counters");
        }
    }
    *out = kv;
    return APEX_OK;
}

void apex_kv_destroy(apex_kv *kv) {
    if (!kv) return;
    for (int i = 0; i < 2; ++i) {
        if (kv->staged[i]) cudaEventDestroy(kv->staged[i]);
        if (kv->staging[i]) cudaFreeHost(kv->staging[i]);
    }
    delete kv;
}

apex_status apex_kv_set_split(apex_kv *kv, int32_t chunk_tokens) {
    if (!kv) return fail(APEX_EINVAL, "kv is NULL");
    if (chunk_tokens < 0 || chunk_tokens % kv->d.block_size)
        return fail(APEX_EINVAL, "chunk_tokens %d must be a non-negative multiple of %d", chunk_tokens,
                    kv->d.block_size);
    kv->forced_chunk_blocks = chunk_tokens / kv->d.block_size;
    return APEX_OK;
}

apex_status apex_kv_set_grid(apex_kv *kv, int32_t ctas) {
    if (!kv || ctas < 0 || ctas > 4 * kv->sm_count) return fail(APEX_EINVAL, "bad grid override");
    kv->grid_override = ctas;
    return APEX_OK;
}

apex_status apex_kv_set_sched(apex_kv *kv, int32_t dyn_permille) {
    if (!kv || dyn_permille < -2 || dyn_permille > 1000)
        return fail(APEX_EINVAL, "dyn_permille %d not in [-2, 1000]", dyn_permille);
    kv->dyn_permille = dyn_permille;
    return APEX_OK;
}

apex_status apex_kv_set_planner(apex_kv *kv, int32_t latency_tiles_per_cta, int32_t guided_div, int32_t guided_pm1,
                                int32_t guided_pm2, int32_t guided_pm3) {
    if (!kv) return fail(APEX_EINVAL, "kv is NULL");
    if (latency_tiles_per_cta < 0 || latency_tiles_per_cta > (1 << 20))
        return fail(APEX_EINVAL, "latency_tiles_per_cta %d not in [0, 2^20]", latency_tiles_per_cta);
    if (guided_div < 1 || guided_div > 64) return fail(APEX_EINVAL, "guided_div %d not in [1, 64]", guided_div);
    if (!(0 <= guided_pm1 && guided_pm1 <= guided_pm2 && guided_pm2 <= guided_pm3 && guided_pm3 <= 1000))
        return fail(APEX_EINVAL, "guided permilles must satisfy 0 <= %d <= %d <= %d <= 1000", guided_pm1, guided_pm2,
                    guided_pm3);
    kv->latency_tiles_per_cta = latency_tiles_per_cta;
    kv->guided[0] = guided_div;
    kv->guided[1] = guided_pm1;
    kv->guided[2] = guided_pm2;
    kv->guided[3] = guided_pm3;
    return APEX_OK;
}

int32_t apex_kv_num_free_blocks(const apex_kv *kv) { return kv ? (int32_t)kv->free_stack.size() : -1; }

int32_t apex_kv_decode_launches(const apex_kv *kv) {
    if (!kv || !kv->have_step) return -1;
    return kv->fuse_merge ? 1 : 2;
}

apex_status apex_kv_seq_info(const apex_kv *kv, int32_t seq_id, int32_t *len, int32_t *blocks, int32_t cap,
                             int32_t *n_blocks) {
    if (!kv) return fail(APEX_EINVAL, "kv is NULL");
    if (seq_id < 0 || seq_id >= kv->d.max_seqs || !kv->seqs[seq_id].live)
        return fail(APEX_ESEQ, "sequence %d is not live", seq_id);
    const auto &s = kv->seqs[seq_id];
    if (len) *len = s.len;
    if (n_blocks) *n_blocks = (int32_t)s.blocks.size();
    if (blocks)
        for (int32_t i = 0; i < std::min<int32_t>(cap, (int32_t)s.blocks.size()); ++i) blocks[i] = s.blocks[i];
    return APEX_OK;
}

apex_status apex_kv_last_slots(const apex_kv *kv, int32_t *slots, int32_t cap, int32_t *n) {
    if (!kv || !kv->have_step) return fail(APEX_EINVAL, "no step allocated");
    if (n) *n = (int32_t)kv->slots.size();
    if (slots)
        for (int32_t i = 0; i < std::min<int32_t>(cap, (int32_t)kv->slots.size()); ++i) slots[i] = kv->slots[i];
    return APEX_OK;
}

apex_status apex_kv_plan_ranges(const apex_kv *kv, int32_t *cta_begin, int32_t cap, int32_t *n) {
    if (!kv || !kv->have_step) return fail(APEX_EINVAL, "no step allocated");
    if (n) *n = (int32_t)kv->cta_begin.size();
    if (cta_begin)
        for (int32_t i = 0; i < std::min<int32_t>(cap, (int32_t)kv->cta_begin.size()); ++i)
            cta_begin[i] = kv->cta_begin[i];
    return APEX_OK;
}

apex_status apex_kv_plan(const apex_kv *kv, int32_t *items, int32_t cap, int32_t *n_items, int32_t *n_merges) {
    if (!kv || !kv->have_step) return fail(APEX_EINVAL, "no step allocated");
    if (n_items) *n_items = (int32_t)kv->items.size();
    if (n_merges) *n_merges = (int32_t)kv->merges.size();
    if (items)
        for (int32_t i = 0; i < std::min<int32_t>(cap, (int32_t)kv->items.size()); ++i) {
            const WorkItem &w = kv->items[i];
            int32_t *o = items + 6 * (size_t)i;
            o[0] = w.b; o[1] = w.g; o[2] = w.blk0; o[3] = w.nblk; o[4] = w.part; o[5] = w.seq;
        }
    return APEX_OK;
}

// Split-KV planner (FlashDecoding lineage).  T = total (block, kv-head)
// tiles, P = persistent CTAs.  Each (row, kv-head) pair is cut into
// near-equal pieces of at most `chunk` blocks; items run longest-first from
// the device queue (greedy LPT on P CTAs).
//  * latency regime (T <= 512 P): chunk from a makespan model (few rounds of
//    near-equal items, whole pairs when cheaper), and the LSE merge is fused
//    into the decode kernel (one launch; the merging CTA's stall is at the end);
//  * bandwidth regime, guided (default): chunk = max(16, ceil(T/8P)), halved /
//    quartered / eighthed for the pairs holding the last 10 / 5 / 2% of the
//    tiles, so the longest-first queue ends with small items; uniform
//    (apex_kv_set_sched(-1)): chunk = max(16, ceil(T/16P)); stream-K ranges
//    (apex_kv_set_sched(>= 0)); pairs shorter than the chunk stay whole;
//  * a forced chunk (apex_kv_set_split) is used as is.
// A pair cut into >1 pieces gets partial slots and a merge entry.
namespace {
void pieces_of(int32_t nblk, int64_t chunk, std::vector<int32_t> &out) {
    out.clear();
    const int32_t n = (int32_t)cdiv(nblk, chunk);
    for (int32_t i = 0; i < n; ++i) out.push_back(nblk / n + (i < nblk % n ? 1 : 0));
}
}  // namespace

// Stream-K variant of the bandwidth regime (apex_kv_set_sched, dyn_permille >= 0):
// the tiles, flattened in (row, kv head, block) order, are dealt out as one
// contiguous static range of ~T_static/P tiles per CTA -- a CTA's range covers
// the tail of one pair, whole pairs and the head of the next, so it runs only a
// few items and never touches the queue; pairs cut at a range boundary are
// merged like any split pair.  The last dyn_permille of the tiles are cut into
// small items (<= 8 per CTA) pulled from the queue by CTAs that finish their
// range early: they absorb SM-to-SM bandwidth differences.
namespace {
struct Piece {
    int32_t cta;    // static owner, or -1 for the dynamic queue
    int32_t blk0, nblk;
};
}  // namespace

static void plan_streamk(const std::vector<int32_t> &nblks, int32_t Hkv, int64_t P, int64_t T, int32_t dyn_permille,
                         std::vector<std::vector<Piece>> &pair_pieces) {
    const int64_t T_dyn = T * dyn_permille / 1000, T_st = T - T_dyn;
    const int64_t dchunk = std::max<int64_t>(16, cdiv(T_dyn, 8 * P));
    const int64_t base = T_st / P, rem = T_st % P;
    auto quota = [&](int64_t c) { return base + (c < rem ? 1 : 0); };
    int64_t c = 0, left = quota(0);
    while (c < P && left == 0) left = quota(++c);
    const int32_t B = (int32_t)nblks.size();
    pair_pieces.assign((size_t)B * Hkv, {});
    std::vector<int32_t> dp;
    for (int32_t b = 0; b < B; ++b)
        for (int32_t g = 0; g < Hkv; ++g) {
            auto &pp = pair_pieces[(size_t)b * Hkv + g];
            int32_t blk = 0, r = nblks[b];
            while (r > 0 && c < P) {
                const int32_t take = (int32_t)std::min<int64_t>(r, left);
                pp.push_back({(int32_t)c, blk, take});
                blk += take;
                r -= take;
                left -= take;
                while (c < P && left == 0) left = quota(++c);
            }
            if (r > 0) {                               // beyond the static share: dynamic pieces
                pieces_of(r, dchunk, dp);
                for (int32_t n : dp) {
                    pp.push_back({-1, blk, n});
                    blk += n;
                }
            }
        }
}

namespace {
// Result of planning one step; committed into the handle only when the whole
// apex_kv_alloc call succeeds (all-or-nothing, include/apex.h).
struct Plan {
    std::vector<WorkItem> items;
    std::vector<MergeItem> merges;
    std::vector<int32_t> cta_begin;
    bool fuse_merge = false;
    int32_t grid = 0;
};
}  // namespace

static apex_status plan_step(const apex_kv *kv, const std::vector<int32_t> &seq_of_row,
                             const std::vector<int32_t> &lens, Plan &out) {
    const int32_t Hkv = kv->d.num_kv_heads, B = (int32_t)lens.size();
    const int64_t P = std::max<int64_t>(1, kv->grid_override > 0
                                               ? kv->grid_override
                                               : apex::decode_grid_ctas(kv->d.dtype, kv->group, kv->sm_count));
    std::vector<int32_t> &nblks = kv->sc.nblks;
    nblks.resize(B);
    int64_t T = 0;

    for (int32_t b = 0; b < B; ++b) {
        nblks[b] = (int32_t)cdiv(lens[b], kv->d.block_size);
        T += (int64_t)nblks[b] * Hkv;

    }
    int64_t chunk = 0;
    bool latency = false, streamk = false;
    if (kv->forced_chunk_blocks > 0) {
        chunk = kv->forced_chunk_blocks;
    } else if (T <= kv->latency_tiles_per_cta * P) {
        // chunk minimising the estimated makespan rounds * (largest piece * t_tile +
        // t_item) over candidate chunks, rounds = ceil(items / P).  ceil(T/P) alone
        // can cut pairs into just more pieces than CTAs (e.g. 128 pairs of 129
        // blocks: chunk 56 -> 384 items, a second round for 88 CTAs: 47 us; chunk
        // 65 -> 256 items: 38 us) or leave 1024 whole pairs at 3.5 rounds.
        // t_tile ~ 0.34 us (8 KiB at a CTA's share of HBM), t_item ~ 3 us (per-item
        // cost incl. the split's merge share; fitted on batch 128 x 512: whole pairs
        // 63.5 us vs halves 70.7 us), in units of 0.01 us.
        // the model depends on the lengths only through their distinct values (counted),
        // and many candidates coincide: evaluate each distinct candidate once over the
        // distinct lengths (host time of a uniform batch-256 plan: ~150 -> ~10 us)
        std::vector<int32_t> &uv = kv->sc.cnt;                 // sorted lengths -> (value, count) pairs
        uv.assign(nblks.begin(), nblks.end());
        std::sort(uv.begin(), uv.end());
        std::vector<std::pair<int32_t, int64_t>> hist;
        for (size_t i = 0; i < uv.size();) {
            size_t j = i;
            while (j < uv.size() && uv[j] == uv[i]) ++j;
            hist.push_back({uv[i], (int64_t)(j - i)});
            i = j;
        }
        const int32_t maxn = std::max<int32_t>(1, hist.back().first);
        auto cost = [&](int64_t c) {
            int64_t n = 0, big = 0;
            for (const auto &h : hist) {
                const int64_t k = cdiv(h.first, c);
                n += k * Hkv * h.second;
                big = std::max(big, cdiv(h.first, k));
            }
            return cdiv(n, P) * (big * 34 + 300);
        };
        std::vector<int64_t> cand;
        for (int64_t k = 1; k <= 64; ++k) cand.push_back(cdiv(maxn, k));
        for (int64_t r = 1; r <= 16; ++r) cand.push_back(std::max<int64_t>(1, cdiv(T, P * r)));
        std::sort(cand.begin(), cand.end(), std::greater<int64_t>());   // larger chunk first: ties keep it
        cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
        int64_t best = -1;
        chunk = maxn;
        for (int64_t c : cand) {
            const int64_t v = cost(c);
            if (best < 0 || v < best || (v == best && c > chunk)) {
                best = v;
                chunk = c;
            }
        }
        latency = true;
    } else if (kv->dyn_permille >= 0) {
        streamk = true;
    } else {
        chunk = std::max<int64_t>(16, cdiv(T, 16 * P));   // >= 16 tiles: per-item costs stay small
    }
    // pieces of every (row, kv head) pair, in pair order -> work items (+ merges of split pairs)
    std::vector<std::vector<WorkItem>> st_items(streamk ? P : 0);
    std::vector<WorkItem> &dyn = kv->sc.dyn;
    std::vector<MergeItem> &merges = out.merges;
    dyn.clear();
    merges.clear();
    int32_t parts = 0;
    size_t n_items = 0;
    auto emit = [&](int32_t b, int32_t g, const Piece *pp, size_t np) {
        const bool split = np > 1;
        const int32_t mg = split ? (int32_t)merges.size() : -1;
        if (split) merges.push_back({b, g, parts, (int32_t)np});
        for (size_t i = 0; i < np; ++i) {
            const WorkItem w{b, g, pp[i].blk0, pp[i].nblk, split ? parts + (int32_t)i : -1, seq_of_row[b], lens[b],
                             mg};
            (pp[i].cta >= 0 ? st_items[pp[i].cta] : dyn).push_back(w);
        }
        if (split) parts += (int32_t)np;
        n_items += np;
    };
    if (streamk) {
        std::vector<std::vector<Piece>> pair_pieces;
        plan_streamk(nblks, Hkv, P, T, kv->dyn_permille, pair_pieces);
        for (int32_t b = 0; b < B; ++b)
            for (int32_t g = 0; g < Hkv; ++g) {
                const auto &pp = pair_pieces[(size_t)b * Hkv + g];
                emit(b, g, pp.data(), pp.size());
            }
    } else {
        std::vector<int32_t> &pc = kv->sc.pc;
        std::vector<Piece> pcs;
        // guided (apex_kv_set_sched(-2)): the pairs holding the last fractions of the
        // tiles (flattened order) are cut into halved, quartered, ... chunks, so the
        // queue (longest first) ends with small items and the CTAs finish together
        const bool guided = !latency && kv->forced_chunk_blocks == 0 && kv->dyn_permille == -2;
        // bulk pieces of T/(g0 P) tiles; the tail pieces halve from T/(max(g0, 8) P), so a
        // small g0 keeps the bulk pairs whole (fewer items and split pairs) while the end of
        // the queue stays as fine as with g0 = 8 (identical plans for g0 >= 8)
        int64_t tail_base = chunk;
        if (guided) {
            chunk = std::max<int64_t>(16, cdiv(T, (int64_t)kv->guided[0] * P));
            tail_base = std::max<int64_t>(16, cdiv(T, (int64_t)std::max<int32_t>(kv->guided[0], 8) * P));
        }
        int64_t pos = 0, last_c = -1;
        int32_t last_n = -1;
        for (int32_t b = 0; b < B; ++b) {
            for (int32_t g = 0; g < Hkv; ++g) {
                if (g == 0 || guided) {
                    int64_t c = chunk;
                    for (int k = 1; guided && k < 4; ++k)
                        if (pos * 1000 >= (int64_t)kv->guided[k] * T) c = std::max<int64_t>(8, tail_base >> k);
                    if (c != last_c || nblks[b] != last_n) {   // pieces depend on (length, chunk) only
                        pieces_of(nblks[b], c, pc);
                        pcs.clear();
                        int32_t blk = 0;
                        for (int32_t n : pc) {
                            pcs.push_back({-1, blk, n});
                            blk += n;
                        }
                        last_c = c;
                        last_n = nblks[b];
                    }
                }
                pos += nblks[b];
                emit(b, g, pcs.data(), pcs.size());
            }
            if ((int64_t)n_items > kv->ws.max_items) break;   // reported below; stop growing
        }
    }
    if ((int64_t)n_items > kv->ws.max_items)
        return fail(APEX_EINVAL, "split chunk of %lld tokens yields %s%zu work items > workspace capacity %d",
                    (long long)chunk * kv->d.block_size, streamk ? "" : "at least ", n_items, kv->ws.max_items);
    std::vector<WorkItem> &items = out.items;
    items.clear();
    items.reserve(n_items);
    out.cta_begin.assign((size_t)P + 1, 0);
    // the dynamic queue longest-first: a stable counting sort on nblk (descending),
    // identical to std::stable_sort with a.nblk > b.nblk, O(items + max nblk)
    std::vector<WorkItem> &sorted = kv->sc.items;
    {
        int32_t mx = 0;
        for (const WorkItem &w : dyn) mx = std::max(mx, w.nblk);
        std::vector<int32_t> &cnt = kv->sc.cnt;
        cnt.assign((size_t)mx + 2, 0);
        for (const WorkItem &w : dyn) ++cnt[(size_t)(mx - w.nblk) + 1];
        for (size_t k = 1; k < cnt.size(); ++k) cnt[k] += cnt[k - 1];
        sorted.resize(dyn.size());
        for (const WorkItem &w : dyn) sorted[(size_t)cnt[(size_t)(mx - w.nblk)]++] = w;
        dyn.swap(sorted);
    }
    if (streamk) {
        for (int64_t c = 0; c < P; ++c) {
            out.cta_begin[c] = (int32_t)items.size();
            items.insert(items.end(), st_items[c].begin(), st_items[c].end());
        }
        out.cta_begin[P] = (int32_t)items.size();
    } else {
        // CTA c starts with item c (no queue round trip on the launch path), then the queue
        for (int64_t c = 0; c <= P; ++c) out.cta_begin[c] = (int32_t)std::min<int64_t>(c, (int64_t)dyn.size());
    }
    items.insert(items.end(), dyn.begin(), dyn.end());
    out.merges.swap(merges);
    out.fuse_merge = latency;
    out.grid = (int32_t)P;
    return APEX_OK;
}

apex_status apex_kv_alloc(apex_kv *kv, const int32_t *seq_ids, const int32_t *n_new, int32_t n, apex_stream stream) {
    if (!kv) return fail(APEX_EINVAL, "kv is NULL");
    if (!seq_ids || !n_new || n < 1 || n > kv->d.max_batch)
        return fail(APEX_EINVAL, "batch of %d sequences not in [1, max_batch=%d]", n, kv->d.max_batch);
    const int32_t bs = kv->d.block_size;
    auto &sc = kv->sc;
    // ---- 1. validate, plan and size the upload on the would-be lengths, before touching
    // any state: every failure below leaves the handle exactly as it was (all-or-nothing)
    if (sc.seen.size() != (size_t)kv->d.max_seqs || sc.stamp == INT32_MAX) {
        sc.seen.assign(kv->d.max_seqs, 0);
        sc.stamp = 0;
    }
    const int32_t stamp = ++sc.stamp;                 // "seen in this call" = seen[s] == stamp
    std::vector<int32_t> &lens = sc.lens;
    lens.resize(n);
    int64_t need = 0, rows = 0;
    for (int32_t i = 0; i < n; ++i) {
        const int32_t s = seq_ids[i], k = n_new[i];
        if (s < 0 || s >= kv->d.max_seqs) return fail(APEX_EINVAL, "seq id %d out of range", s);
        if (sc.seen[s] == stamp) return fail(APEX_EINVAL, "seq id %d repeated in one alloc", s);
        sc.seen[s] = stamp;
        if (k < 0) return fail(APEX_EINVAL, "n_new[%d] = %d < 0", i, k);
        const int64_t L = kv->seqs[s].live ? kv->seqs[s].len : 0;
        if (L + k < 1) return fail(APEX_EINVAL, "seq %d would have an empty context (reading c4)", s);
        if (L + k > (int64_t)kv->d.max_blocks_per_seq * bs)
            return fail(APEX_EINVAL, "seq %d would exceed max context %d", s, kv->d.max_blocks_per_seq * bs);
        need += cdiv(L + k, bs) - cdiv(L, bs);
        rows += k;
        lens[i] = (int32_t)(L + k);
    }
    if (rows > kv->d.max_new_tokens)
        return fail(APEX_EINVAL, "%lld new tokens > max_new_tokens %d", (long long)rows, kv->d.max_new_tokens);
    if (need > (int64_t)kv->free_stack.size())
        return fail(APEX_ENOBLOCKS, "need %lld blocks, %zu free", (long long)need, kv->free_stack.size());
    std::vector<int32_t> &seq_of_row = sc.seq_of_row;
    seq_of_row.assign(seq_ids, seq_ids + n);
    // the plan is built in spare storage kept by the handle; whatever the exit path, the
    // storage that is not committed goes back to the spares (no per-step allocations)
    Plan plan;
    plan.items.swap(sc.plan_items);
    plan.merges.swap(sc.merges);
    plan.cta_begin.swap(sc.cta_begin);
    struct Spares {
        apex_kv::Scratch &sc;
        Plan &p;
        ~Spares() {
            sc.plan_items.swap(p.items);
            sc.merges.swap(p.merges);
            sc.cta_begin.swap(p.cta_begin);
        }
    } spares{sc, plan};
    apex_status st = plan_step(kv, seq_of_row, lens, plan);
    if (st != APEX_OK) return st;
    // packed upload: header | cta_begin | items (fixed offset) | merges | slots | bt deltas |
    // len deltas -- exactly the used bytes, moved by one upload (the zero-copy upload kernel, or
    // an H2D copy with -DAPEX_UPLOAD_KERNEL=0); kernels find the merge list and the slot map
    // through offsets in the header (fixed launch parameters)
    const size_t items_bytes = sizeof(apex::ItemRec) * plan.items.size();
    const size_t merges_bytes = sizeof(MergeItem) * plan.merges.size();
    const size_t o_merges = align_up(kv->ws.o_items + items_bytes, 256);
    const size_t o_slots = o_merges + align_up(merges_bytes, 256);
    const size_t o_bt = o_slots + align_up(sizeof(int32_t) * (size_t)rows, 256);
    const size_t o_len = o_bt + align_up(sizeof(int2) * (size_t)need, 256);
    const size_t up_end = o_len + align_up(sizeof(int2) * (size_t)n, 256);
    if (!kv->host_only && up_end > kv->ws.upload_cap)
        return fail(APEX_EINVAL, "step metadata (%zu B) exceeds the upload region (%zu B)", up_end, kv->ws.upload_cap);
    const int r = kv->ring;
    if (!kv->host_only && kv->staged_pending[r]) {
        cudaError_t e = cudaEventSynchronize(kv->staged[r]);   // its previous upload must be done
        if (e != cudaSuccess) return cuda_fail(e, "apex_kv_alloc: staging reuse");
        kv->staged_pending[r] = false;
    }

    // ---- 2. commit: pop blocks, compute slots and deltas (cannot fail)
    std::vector<int32_t> &slots = sc.slots;
    slots.clear();
    slots.reserve(rows);
    std::vector<int2> &bt_delta = sc.bt_delta, &len_delta = sc.len_delta;
    bt_delta.clear();
    len_delta.clear();
    std::vector<int32_t> &popped = sc.popped;          // pop order (for the CUDA-failure rollback)
    popped.clear();
    std::vector<apex_kv::Seq> &before = sc.before;     // (live, len) of each seq before the call
    if (before.size() < (size_t)n) before.resize(n);
    for (int32_t i = 0; i < n; ++i) {
        auto &sq = kv->seqs[seq_ids[i]];
        before[i].live = sq.live;
        before[i].len = sq.len;
        if (!sq.live) {
            sq.live = true;
            sq.len = 0;
            sq.blocks.clear();
        }
        for (int32_t pos = sq.len; pos < sq.len + n_new[i]; ++pos) {
            if (pos % bs == 0) {
                const int32_t blk = kv->free_stack.back();
                kv->free_stack.pop_back();
                popped.push_back(blk);
                bt_delta.push_back({seq_ids[i] * kv->d.max_blocks_per_seq + pos / bs, blk});
                sq.blocks.push_back(blk);
            }
            slots.push_back(sq.blocks[pos / bs] * bs + pos % bs);
        }
        sq.len += n_new[i];
        len_delta.push_back({seq_ids[i], sq.len});
    }
    auto rollback = [&] {
        for (int32_t i = n - 1; i >= 0; --i) {
            auto &sq = kv->seqs[seq_ids[i]];
            const size_t nb = (size_t)cdiv(before[i].len, bs);
            sq.blocks.resize(before[i].live ? nb : 0);
            sq.len = before[i].len;
            sq.live = before[i].live;
        }
        for (auto it = popped.rbegin(); it != popped.rend(); ++it) kv->free_stack.push_back(*it);
    };
    if (!kv->host_only) {
        // ---- 3. pack the step metadata into pinned staging and upload it
        uint8_t *host = kv->staging[r];
        apex::StepHeader hdr{};
        hdr.n_items = (int32_t)plan.items.size();
        hdr.n_merges = (int32_t)plan.merges.size();
        hdr.n_rows = (int32_t)rows;
        hdr.o_merges = (int32_t)o_merges;
        hdr.o_slots = (int32_t)o_slots;
        std::memcpy(host, &hdr, sizeof hdr);
        std::memcpy(host + apex::kCtaBeginOffset, plan.cta_begin.data(), sizeof(int32_t) * plan.cta_begin.size());
        // items + the physical ids of their first blocks (known now that the blocks are popped)
        apex::ItemRec *rec = reinterpret_cast<apex::ItemRec *>(host + kv->ws.o_items);
        for (size_t t = 0; t < plan.items.size(); ++t) {
            const WorkItem &it = plan.items[t];
            const std::vector<int32_t> &blocks = kv->seqs[it.seq].blocks;
            rec[t].it = it;
            for (int u = 0; u < apex::kInlineIds; ++u)
                rec[t].ids[u] = u < it.nblk ? blocks[(size_t)it.blk0 + u] : -1;
        }
        if (merges_bytes) std::memcpy(host + o_merges, plan.merges.data(), merges_bytes);
        if (rows) std::memcpy(host + o_slots, slots.data(), sizeof(int32_t) * slots.size());
        if (need) std::memcpy(host + o_bt, bt_delta.data(), sizeof(int2) * bt_delta.size());
        std::memcpy(host + o_len, len_delta.data(), sizeof(int2) * len_delta.size());
        uint8_t *dev = (uint8_t *)kv->d.workspace + kv->ws.upload;
        cudaStream_t s = (cudaStream_t)stream;
#if APEX_UPLOAD_KERNEL
        // ONE launch: copy the metadata from the mapped staging buffer into the device
        // upload region and apply the table / length deltas from the same host copy
        // (an H2D copy + the delta kernel cost two serialised operations per step)
        const uint8_t *hdev = kv->staging_dev[r];
        cudaError_t e = apex::launch_upload(hdev, dev, up_end, (const int2 *)(hdev + o_bt), (int)bt_delta.size(),
                                            (const int2 *)(hdev + o_len), (int)len_delta.size(), kv->d.block_table,
                                            kv->d.seq_lens, kv->sm_count, s);
        if (e == cudaSuccess) e = cudaEventRecord(kv->staged[r], s);
        if (e == cudaSuccess) kv->staged_pending[r] = true;
#else
        cudaError_t e = cudaMemcpyAsync(dev, host, up_end, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) e = cudaEventRecord(kv->staged[r], s);
        if (e == cudaSuccess) {
            kv->staged_pending[r] = true;
            e = apex::launch_apply_deltas((const int2 *)(dev + o_bt), (int)bt_delta.size(),
                                          (const int2 *)(dev + o_len), (int)len_delta.size(), kv->d.block_table,
                                          kv->d.seq_lens, s);
        }
#endif
        if (e != cudaSuccess) {
            rollback();
            // the device header may already hold the withdrawn step: append/decode are
            // refused until the next successful alloc
            kv->have_step = false;
            return cuda_fail(e, "apex_kv_alloc: metadata upload");
        }
        kv->ring ^= 1;
    }
    kv->batch_seq.swap(seq_of_row);
    kv->slots.swap(slots);
    kv->items.swap(plan.items);
    kv->merges.swap(plan.merges);
    kv->cta_begin.swap(plan.cta_begin);
    kv->fuse_merge = plan.fuse_merge;
    kv->plan_grid = plan.grid;
    kv->batch = n;
    kv->n_rows = (int32_t)rows;
    kv->have_step = true;
    kv->single_token_step = true;
    for (int32_t i = 0; i < n; ++i) kv->single_token_step = kv->single_token_step && n_new[i] == 1;
    return APEX_OK;
}

apex_status apex_kv_release(apex_kv *kv, int32_t seq_id) {
    if (!kv) return fail(APEX_EINVAL, "kv is NULL");
    if (seq_id < 0 || seq_id >= kv->d.max_seqs || !kv->seqs[seq_id].live)
        return fail(APEX_ESEQ, "sequence %d is not live", seq_id);
    auto &sq = kv->seqs[seq_id];
    for (auto it = sq.blocks.rbegin(); it != sq.blocks.rend(); ++it) kv->free_stack.push_back(*it);
    sq = apex_kv::Seq();
    return APEX_OK;
}

apex_status apex_kv_append(apex_kv *kv, int32_t layer, const void *k_new, const void *v_new, apex_stream stream) {
    if (!kv) return fail(APEX_EINVAL, "kv is NULL");
    if (kv->host_only) return fail(APEX_EINVAL, "host-only handle has no device pools");
    if (!kv->have_step) return fail(APEX_EINVAL, "apex_kv_append before apex_kv_alloc");
    if (layer < 0 || layer >= kv->d.num_layers) return fail(APEX_EINVAL, "layer %d out of range", layer);
    if (kv->n_rows > 0 && (!k_new || !v_new)) return fail(APEX_EINVAL, "k_new/v_new is NULL");
    if (((uintptr_t)k_new | (uintptr_t)v_new) & 15) return fail(APEX_EINVAL, "k_new/v_new not 16-byte aligned");
    // always one launch (it reads the row count from the step header): graph-capturable
    uint8_t *up = (uint8_t *)kv->d.workspace + kv->ws.upload;
    cudaError_t e = apex::launch_append(kv->d.dtype, k_new, v_new, kv->kv_pools[layer],
                                        nullptr, (const apex::StepHeader *)up,
                                        kv->d.num_kv_heads, kv->sm_count, (cudaStream_t)stream);
    return e == cudaSuccess ? APEX_OK : cuda_fail(e, "apex_kv_append");
}

apex_status apex_decode_attention(apex_kv *kv, int32_t layer, const void *q, void *out, float scale,
                                  apex_stream stream) {
    if (!kv) return fail(APEX_EINVAL, "kv is NULL");
    void *outs[1] = {out};
    return apex_decode_attention_ex(kv, layer, q, outs, 1, (int64_t)kv->d.num_q_heads * kv->d.head_dim,
                                    kv->d.head_dim, 0, nullptr, 0, 0, scale, stream);
}

}  // extern "C"

static apex_status decode_impl(apex_kv *kv, int32_t layer, const void *q, const void *k_new, const void *v_new,
                               void *const *outs, int32_t n_out, int64_t out_row_stride, int64_t out_head_stride,
                               int32_t out_head_offset, uint32_t *const *signals, int32_t signal_slot,
                               uint32_t signal_value, float scale, apex_stream stream) {
    if (!kv) return fail(APEX_EINVAL, "kv is NULL");
    if (kv->host_only) return fail(APEX_EINVAL, "host-only handle has no device pools");
    if (!kv->have_step) return fail(APEX_EINVAL, "apex_decode_attention before apex_kv_alloc");
    if (layer < 0 || layer >= kv->d.num_layers) return fail(APEX_EINVAL, "layer %d out of range", layer);
    if (!q || !outs || n_out < 1 || n_out > apex::kMaxOut)
        return fail(APEX_EINVAL, "q/outs is NULL or n_out %d not in [1, %d]", n_out, apex::kMaxOut);
    // every (row, head) of the step owns a disjoint D-vector of each destination:
    // row-major-like (row stride covers all heads) or head-major-like (head stride
    // covers all rows), strides multiples of 4 elements (8/16-byte vector stores)
    const int64_t D = kv->d.head_dim, H = (int64_t)out_head_offset + kv->d.num_q_heads, B = kv->batch;
    const bool row_major = out_head_stride >= D && out_row_stride >= H * out_head_stride;
    const bool head_major = out_row_stride >= D && out_head_stride >= B * out_row_stride;
    if (out_head_offset < 0 || out_row_stride % 4 || out_head_stride % 4 || !(row_major || head_major))
        return fail(APEX_EINVAL,
                    "out strides (row %lld, head %lld) / head offset %d: rows and heads of the %lld x %lld "
                    "destination must not overlap",
                    (long long)out_row_stride, (long long)out_head_stride, out_head_offset, (long long)B,
                    (long long)H);
    if (signals) {
        if (signal_slot < 0) return fail(APEX_EINVAL, "signal_slot %d < 0", signal_slot);
        for (int32_t i = 0; i < n_out; ++i)
            if (!signals[i] || ((uintptr_t)signals[i] & 3))
                return fail(APEX_EINVAL, "signals[%d] NULL or not 4-byte aligned", i);
    }
    if ((uintptr_t)q & 15) return fail(APEX_EINVAL, "q not 16-byte aligned");
    for (int32_t i = 0; i < n_out; ++i)
        if (!outs[i] || ((uintptr_t)outs[i] & 15)) return fail(APEX_EINVAL, "outs[%d] NULL or not 16-byte aligned", i);
    if (!(scale > 0.0f) || !std::isfinite(scale)) return fail(APEX_EINVAL, "scale must be finite and > 0");
    apex::DecodeParams p{};
    p.q = q;
    for (int32_t i = 0; i < n_out; ++i) p.out[i] = outs[i];
    p.n_out = n_out;
    p.out_row_stride = out_row_stride;
    p.out_head_stride = out_head_stride;
    p.out_head_offset = out_head_offset;
    if (signals)
        for (int32_t i = 0; i < n_out; ++i) p.signals[i] = signals[i];
    p.signal_slot = signal_slot;
    p.signal_value = signal_value;
    p.block_table = kv->d.block_table;
    uint8_t *ws = (uint8_t *)kv->d.workspace;
    uint8_t *up = ws + kv->ws.upload;
    p.hdr = (const apex::StepHeader *)up;
    p.cta_begin = (const int32_t *)(up + apex::kCtaBeginOffset);
    p.items = (const apex::ItemRec *)(up + kv->ws.o_items);
    p.merges = nullptr;                 // device side: hdr->o_merges (packed upload)
    p.part_o = (float *)(ws + kv->ws.part_o);
    p.part_ml = (float *)(ws + kv->ws.part_ml);
    p.counters = (int32_t *)(ws + kv->ws.counters) + 2 * layer;
    p.sig_counter = (int32_t *)(ws + kv->ws.counters) + 2 * apex::kMaxLayers + layer;
    p.merge_counters = (int32_t *)(ws + kv->ws.merge_counters);
    p.merge_grid = (int32_t)std::max<int64_t>(1, std::min<int64_t>(kv->ws.max_merges, 16LL * kv->sm_count));
    p.max_blocks_per_seq = kv->d.max_blocks_per_seq;
    p.num_q_heads = kv->d.num_q_heads;
    p.num_kv_heads = kv->d.num_kv_heads;
    p.scale_log2 = (float)((double)scale * 1.4426950408889634);   // log2(e)
    p.tma_segs = kv->tma_segs;
    p.fuse_merge = kv->fuse_merge ? 1 : 0;
    if (k_new) {
        if (!v_new || (((uintptr_t)k_new | (uintptr_t)v_new) & 15))
            return fail(APEX_EINVAL, "k_new/v_new NULL or not 16-byte aligned");
        if (!kv->single_token_step)
            return fail(APEX_EINVAL, "fused append needs exactly one new token per sequence in the step "
                                     "(use apex_kv_append + apex_decode_attention)");
        if (kv->fuse_merge) {
            // latency regime: the append rides in the decode launch (one launch per call)
            p.k_new = k_new;
            p.v_new = v_new;
            p.kv_pool = kv->kv_pools[layer];
            p.num_blocks = kv->d.num_blocks;
        } else {
            // bandwidth regime: the separate append kernel + the plain decode kernel is
            // faster than the fused-append decode kernel (whose per-tile checks and row
            // patch cost 2-6% of a 4-64 GiB stream, more than the saved launch)
            uint8_t *up = (uint8_t *)kv->d.workspace + kv->ws.upload;
            cudaError_t e = apex::launch_append(kv->d.dtype, k_new, v_new, kv->kv_pools[layer],
                                                nullptr, (const apex::StepHeader *)up,
                                                kv->d.num_kv_heads, kv->sm_count, (cudaStream_t)stream);
            if (e != cudaSuccess) return cuda_fail(e, "apex_decode_attention_append (append)");
        }
    }
    // fixed persistent grid (CTAs without an item exit at once): every launch parameter is
    // step-invariant, so the per-layer launches can be captured in a CUDA graph
    const int grid = kv->plan_grid;   // cta_begin has plan_grid + 1 entries
    cudaError_t e = apex::launch_decode(kv->d.dtype, kv->group, kv->tmaps[layer], p, grid, (cudaStream_t)stream);
    return e == cudaSuccess ? APEX_OK : cuda_fail(e, "apex_decode_attention");
}

extern "C" {

apex_status apex_decode_attention_ex(apex_kv *kv, int32_t layer, const void *q, void *const *outs, int32_t n_out,
                                     int64_t out_row_stride, int64_t out_head_stride, int32_t out_head_offset,
                                     uint32_t *const *signals, int32_t signal_slot, uint32_t signal_value,
                                     float scale, apex_stream stream) {
    return decode_impl(kv, layer, q, nullptr, nullptr, outs, n_out, out_row_stride, out_head_stride, out_head_offset,
                       signals, signal_slot, signal_value, scale, stream);
}

apex_status apex_decode_attention_append(apex_kv *kv, int32_t layer, const void *q, const void *k_new,
                                         const void *v_new, void *out, float scale, apex_stream stream) {
    if (!kv) return fail(APEX_EINVAL, "kv is NULL");
    if (!k_new || !v_new) return fail(APEX_EINVAL, "k_new/v_new is NULL");
    void *outs[1] = {out};
    return decode_impl(kv, layer, q, k_new, v_new, outs, 1, (int64_t)kv->d.num_q_heads * kv->d.head_dim,
                       kv->d.head_dim, 0, nullptr, 0, 0, scale, stream);
}

apex_status apex_signal_wait(const uint32_t *signals, int32_t n, uint32_t value, uint64_t timeout_ns,
                             uint32_t *status, apex_stream stream) {
    if (!signals || n < 1 || ((uintptr_t)signals & 3))
        return fail(APEX_EINVAL, "apex_signal_wait: signals NULL/misaligned or n %d < 1", n);
    if (status && ((uintptr_t)status & 3)) return fail(APEX_EINVAL, "apex_signal_wait: status misaligned");
    cudaError_t e = apex::launch_signal_wait(signals, n, value, timeout_ns, status, (cudaStream_t)stream);
    return e == cudaSuccess ? APEX_OK : cuda_fail(e, "apex_signal_wait");
}

apex_status apex_signal_post(uint32_t *const *dst, int32_t n_dst, int32_t slot, uint32_t value, apex_stream stream) {
    if (!dst || n_dst < 1 || n_dst > apex::kMaxOut || slot < 0)
        return fail(APEX_EINVAL, "apex_signal_post: dst NULL, n_dst %d not in [1, %d] or slot %d < 0", n_dst,
                    apex::kMaxOut, slot);
    for (int32_t i = 0; i < n_dst; ++i)
        if (!dst[i] || ((uintptr_t)dst[i] & 3)) return fail(APEX_EINVAL, "apex_signal_post: dst[%d] NULL/misaligned", i);
    cudaError_t e = apex::launch_signal_post(dst, n_dst, slot, value, (cudaStream_t)stream);
    return e == cudaSuccess ? APEX_OK : cuda_fail(e, "apex_signal_post");
}

// ---------------------------------------------------------------- cost model

}  // extern "C"

struct apex_cost {
    std::vector<double> batch, kv, us;   // us[i * nk + j]
};

namespace {
constexpr size_t kMaxCostGrid = 256;     // grid points per axis (apex_cost_observe may add lines)
}

namespace {
// (cell, fraction) of x on a strictly increasing grid, clamped to its ends
void locate(const std::vector<double> &g, double x, size_t &i, double &f) {
    if (g.size() == 1 || x <= g.front()) { i = 0; f = 0.0; return; }
    if (x >= g.back()) { i = g.size() - 2; f = 1.0; return; }
    i = (size_t)(std::upper_bound(g.begin(), g.end(), x) - g.begin()) - 1;
    f = (x - g[i]) / (g[i + 1] - g[i]);
}
}  // namespace

extern "C" {

apex_status apex_cost_create(const int32_t *batch, int32_t nb, const int64_t *kv_tokens, int32_t nk,
                             const double *us, apex_cost **out) {
    if (!out) return fail(APEX_EINVAL, "out is NULL");
    *out = nullptr;
    if (!batch || !kv_tokens || !us || nb < 1 || nk < 1) return fail(APEX_EINVAL, "empty cost table");
    for (int32_t i = 0; i < nb; ++i)
        if (batch[i] <= 0 || (i && batch[i] <= batch[i - 1]))
            return fail(APEX_EINVAL, "batch grid must be positive and strictly increasing (entry %d)", i);
    for (int32_t j = 0; j < nk; ++j)
        if (kv_tokens[j] <= 0 || (j && kv_tokens[j] <= kv_tokens[j - 1]))
            return fail(APEX_EINVAL, "kv_tokens grid must be positive and strictly increasing (entry %d)", j);
    for (int64_t i = 0; i < (int64_t)nb * nk; ++i)
        if (!std::isfinite(us[i]) || us[i] <= 0.0) return fail(APEX_EINVAL, "time entry %lld not finite/positive", (long long)i);
    apex_cost *c = new (std::nothrow) apex_cost();
    if (!c) return fail(APEX_EINVAL, "out of host memory");
    c->batch.assign(batch, batch + nb);
    c->kv.assign(kv_tokens, kv_tokens + nk);
    c->us.assign(us, us + (size_t)nb * nk);
    *out = c;
    return APEX_OK;
}

apex_status apex_predict_time(const apex_cost *c, int32_t batch, int64_t kv_tokens, double *us_out) {
    if (!c || !us_out) return fail(APEX_EINVAL, "cost/us_out is NULL");
    size_t i, j;
    double fx, fy;
    locate(c->batch, (double)batch, i, fx);
    locate(c->kv, (double)kv_tokens, j, fy);
    const size_t nk = c->kv.size();
    const size_t i1 = std::min(i + 1, c->batch.size() - 1), j1 = std::min(j + 1, nk - 1);
    const double u00 = c->us[i * nk + j], u10 = c->us[i1 * nk + j];
    const double u01 = c->us[i * nk + j1], u11 = c->us[i1 * nk + j1];
    *us_out = (1 - fx) * (1 - fy) * u00 + fx * (1 - fy) * u10 + (1 - fx) * fy * u01 + fx * fy * u11;
    return APEX_OK;
}

// Online recalibration (§6; reading c17): grid lines through an
// outside point (valued at the current clamped predictions, so no prediction changes),
// then a normalised LMS step on the point's cell corners: prediction at the point
// becomes exactly predicted + alpha * (measured - predicted).
apex_status apex_cost_observe(apex_cost *c, int32_t batch, int64_t kv_tokens, double measured_us, double alpha) {
    if (!c) return fail(APEX_EINVAL, "cost is NULL");
    if (!(alpha > 0.0 && alpha <= 1.0)) return fail(APEX_EINVAL, "alpha %g not in (0, 1]", alpha);
    if (!std::isfinite(measured_us) || measured_us <= 0.0)
        return fail(APEX_EINVAL, "measured_us %g must be finite and > 0", measured_us);
    const double x = (double)batch, y = (double)kv_tokens;
    const bool out_x = x < c->batch.front() || x > c->batch.back();
    const bool out_y = y < c->kv.front() || y > c->kv.back();
    if ((out_x && c->batch.size() >= kMaxCostGrid) || (out_y && c->kv.size() >= kMaxCostGrid))
        return fail(APEX_EINVAL, "cost grid is full (%d points per axis)", kMaxCostGrid);
    apex_cost n = *c;   // work on a copy: all-or-nothing
    double pred = 0.0;
    if (out_x) {
        const size_t nk = n.kv.size(), at = x < n.batch.front() ? 0 : n.batch.size();
        std::vector<double> row(nk);
        for (size_t j = 0; j < nk; ++j) apex_predict_time(&n, batch, (int64_t)n.kv[j], &row[j]);
        n.batch.insert(n.batch.begin() + at, x);
        n.us.insert(n.us.begin() + at * nk, row.begin(), row.end());
    }
    if (out_y) {
        const size_t nb = n.batch.size(), nk = n.kv.size(), at = y < n.kv.front() ? 0 : nk;
        std::vector<double> col(nb), us;
        for (size_t i = 0; i < nb; ++i) apex_predict_time(&n, (int32_t)n.batch[i], kv_tokens, &col[i]);
        us.reserve(nb * (nk + 1));
        for (size_t i = 0; i < nb; ++i) {
            us.insert(us.end(), n.us.begin() + i * nk, n.us.begin() + i * nk + at);
            us.push_back(col[i]);
            us.insert(us.end(), n.us.begin() + i * nk + at, n.us.begin() + (i + 1) * nk);
        }
        n.kv.insert(n.kv.begin() + at, y);
        n.us.swap(us);
    }
    apex_predict_time(&n, batch, kv_tokens, &pred);
    const double e = measured_us - pred;
    size_t i, j;
    double fx, fy;
    locate(n.batch, x, i, fx);
    locate(n.kv, y, j, fy);
    const size_t nk = n.kv.size();
    const size_t i1 = std::min(i + 1, n.batch.size() - 1), j1 = std::min(j + 1, nk - 1);
    // corners with their bilinear weights; coincident corners (1-point axis) merged
    size_t idx[4] = {i * nk + j, i1 * nk + j, i * nk + j1, i1 * nk + j1};
    double w[4] = {(1 - fx) * (1 - fy), fx * (1 - fy), (1 - fx) * fy, fx * fy};
    for (int a = 0; a < 4; ++a)
        for (int b = 0; b < a; ++b)
            if (idx[b] == idx[a] && w[a] != 0.0) {
                w[b] += w[a];
                w[a] = 0.0;
            }
    double norm = 0.0;
    for (int a = 0; a < 4; ++a) norm += w[a] * w[a];
    for (int a = 0; a < 4; ++a)
        if (w[a] != 0.0) n.us[idx[a]] += alpha * e * w[a] / norm;
    *c = std::move(n);
    return APEX_OK;
}

apex_status apex_cost_size(const apex_cost *c, int32_t *nb, int32_t *nk) {
    if (!c) return fail(APEX_EINVAL, "cost is NULL");
    if (nb) *nb = (int32_t)c->batch.size();
    if (nk) *nk = (int32_t)c->kv.size();
    return APEX_OK;
}

apex_status apex_cost_table(const apex_cost *c, int32_t *batch, int64_t *kv_tokens, double *us) {
    if (!c) return fail(APEX_EINVAL, "cost is NULL");
    if (batch)
        for (size_t i = 0; i < c->batch.size(); ++i) batch[i] = (int32_t)c->batch[i];
    if (kv_tokens)
        for (size_t j = 0; j < c->kv.size(); ++j) kv_tokens[j] = (int64_t)c->kv[j];
    if (us) std::memcpy(us, c->us.data(), sizeof(double) * c->us.size());
    return APEX_OK;
}

void apex_cost_destroy(apex_cost *c) { delete c; }

}  // extern "C"
