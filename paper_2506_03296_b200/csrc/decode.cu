// Split-KV paged decode attention for sm_100a (B200).
//
// Computes, per work item (batch row b, kv head g, logical blocks [blk0, blk0+nblk)),
// the online-softmax partial of  softmax(scale * q . K^T) . V  for the g-th
// q-group (PAPER.md P:49-53 decode attention, P:51 GQA sharing, P:79
// memory-bound; FlashDecoding-style split + log-sum-exp merge, cited at P:53).
//
// Kernel design:
//  * persistent grid, 2 CTAs/SM; CTA i starts with item i, then pulls items
//    longest-first from a device work queue (atomicAdd), so ragged contexts
//    balance across the 148 SMs;
//  * warp 0 = producer: reads the block table 32 entries at a time and issues
//    one TMA (cp.async.bulk.tensor, 128-B swizzle) per (block, kv-head) tile --
//    its 16 K rows and 16 V rows, contiguous in the interleaved pool: 8 KiB
//    (16-bit) / 16 KiB (fp32) -- into mbarrier-guarded shared-memory slots;
//  * warps 1..4 = consumers: tile j of an item goes to consumer j % 4, each
//    keeps its own running (m, l, O) and the four are merged through shared
//    memory at the item's end (fixed order => deterministic).  Every consumer
//    owns a private sub-ring of SW slots that it waits on strictly in order:
//    with one shared ring a fast warp could wait on a slot whose previous fill
//    was still in flight, and mbarrier try_wait.parity would report the
//    preceding phase as complete (a race seen at C2 sizes);
//  * GQA (g >= 2, 16-bit): S^T = K Q_g^T and O^T += V^T P^T on tensor cores with
//    mma.sync.m16n8k16, the q-group on the N = 8 side (16 HMMA per 16-token
//    tile), K/V fragments via ldmatrix(.trans) on the swizzled tiles
//    (conflict-free), P^T re-laid from the S^T accumulators by movmatrix.trans;
//  * fp32 (MHA): CUDA-core FMAs, one lane per token for q.K (conflict-free
//    thanks to the swizzle), lane-owned dims for P.V; 16-bit MHA uses the
//    tensor-core path above with one live head column (fewer instructions).
//  * softmax in the log2 domain (scale*log2e folded into S); split items write
//    (m, l, unnormalised O) fp32 partials merged in split order -- by a second
//    small launch (fixed grid, grid-stride over split pairs) in the bandwidth
//    regime, or, in the latency regime, by the last split of the pair to finish
//    (per-pair arrival counter) inside this kernel, saving the launch;
//  * every launch parameter is step-invariant (counts from the device step
//    header, fixed grids), so the launches are CUDA-graph capturable, and they
//    use programmatic dependent launch (griddepcontrol) to overlap prologues.
#include <type_traits>

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "apex_internal.h"

namespace apex {
#ifdef APEX_TRACE
// timing instrumentation (tuning builds only): globaltimer stamps per CTA
__device__ unsigned long long g_apex_trace[1024][16];
__device__ __forceinline__ void trace(int ev) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x < 1024) g_apex_trace[blockIdx.x][ev] = t;
}
__device__ __forceinline__ void trace_val(int ev, unsigned long long v) {
    if (blockIdx.x < 1024) g_apex_trace[blockIdx.x][ev] = v;
}
#define TRACE(ev) trace(ev)
#define TRACE_VAL(ev, v) trace_val(ev, v)
#else
#define TRACE(ev) ((void)0)
#define TRACE_VAL(ev, v) ((void)0)
#endif
namespace {

#ifndef APEX_NC
#define APEX_NC 4
#endif
#ifndef APEX_CTAS_PER_SM
#define APEX_CTAS_PER_SM 2
#endif
#ifndef APEX_SPEC_ITEM
#define APEX_SPEC_ITEM 1
#endif
#ifndef APEX_MSCR_ALL
#define APEX_MSCR_ALL 0
#endif
#ifndef APEX_Q_LDG
#define APEX_Q_LDG 0
#endif
#if APEX_Q_LDG
#define LDQ(p) __ldg(p)
#else
#define LDQ(p) (*(p))
#endif
#ifndef APEX_MERGE_UNROLL
#define APEX_MERGE_UNROLL 16
#endif
#ifndef APEX_MAX_SLOTS
#define APEX_MAX_SLOTS 24
#endif
#ifndef APEX_L2_EVICT_FIRST
#define APEX_L2_EVICT_FIRST 0
#endif
constexpr int NC = APEX_NC;              // consumer warps
constexpr int NTHREADS = 32 * (NC + 1);   // producer warp + NC consumer warps
constexpr int IR = 4;                    // item-ring entries
constexpr int CTAS_PER_SM = APEX_CTAS_PER_SM;
constexpr int kMergeUnroll = APEX_MERGE_UNROLL;   // parts in flight per thread in the LSE merge
constexpr int kTileRows = kBlock;        // 16 tokens per tile
// smem tile of one (block, kv head): [segment][32 rows: K 0-15, V 16-31][128 B], 128-B swizzled
constexpr int kSegStride = 2 * kTileRows * 128;
constexpr int kVOff = kTileRows * 128;

struct ItemSlot {
    WorkItem it;
    int32_t pad[4];
};

constexpr int kSmemPerCta = (232448 - 1024 * CTAS_PER_SM) / CTAS_PER_SM - 1024;   // SM carve-out split

template <int DT, int G, bool FUSE = true> struct Cfg {
    static constexpr int ES = DT == APEX_F32 ? 4 : 2;
    static constexpr int TILE = kTileRows * kHeadDim * ES;   // bytes of the K (or the V) half of a tile
    static constexpr int CB_O = NC * G * kHeadDim * 4;       // per-warp O for the item merge
    static constexpr int CB_ML = NC * G * 2 * 4 + 16;     // + merge flag
    static constexpr int MSCR = (FUSE || APEX_MSCR_ALL) ? NC * 32 * (16 + 8) : 0;   // fused merge: red + redml per thread
    static constexpr int RING = IR * (int)sizeof(ItemSlot);
    static constexpr int FIXED = CB_O + CB_ML + MSCR + RING + 2 * IR * 8 + 1024;
    static constexpr int S0 = (kSmemPerCta - FIXED) / (2 * TILE + 16);
    static constexpr int SW = (S0 > APEX_MAX_SLOTS ? APEX_MAX_SLOTS : S0) / NC;   // slots per consumer warp
    static constexpr int STAGES = SW * NC;
    static constexpr int TILES = STAGES * 2 * TILE;
    static constexpr int BARS = (2 * STAGES + 2 * IR) * 8;
    static constexpr int TOTAL = TILES + BARS + RING + CB_O + CB_ML + MSCR + 1024;   // + alignment slack
    static_assert(TOTAL <= kSmemPerCta, "shared memory budget");
    static_assert(SW >= 1, "ring too shallow");
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap *map, uint32_t bar, int c0, int c1,
                                            int c2) {
#if APEX_L2_EVICT_FIRST
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
        : "memory");
#else
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
#endif
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, uint32_t bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// exp2(x - m) that is exactly 1 when x == m (ctx=1 and max-token bit-exactness)
__device__ __forceinline__ float ex2_diff(float x, float m) { return x == m ? 1.0f : ex2(x - m); }

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr));
    return v;
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
// 16-bit pair <-> floats
template <int DT> __device__ __forceinline__ float2 unpack2(uint32_t u) {
    if constexpr (DT == APEX_BF16) {
        return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xffff0000u));
    } else {
        __half2 h = *reinterpret_cast<__half2 *>(&u);
        return __half22float2(h);
    }
}
template <int DT> __device__ __forceinline__ uint32_t pack2(float lo, float hi) {
    if constexpr (DT == APEX_BF16) {
        __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
        return *reinterpret_cast<uint32_t *>(&v);
    } else {
        __half2 v = __floats2half2_rn(lo, hi);
        return *reinterpret_cast<uint32_t *>(&v);
    }
}
template <int DT> __device__ __forceinline__ void store4(void *out, size_t idx, float a, float b, float c, float d) {
    if constexpr (DT == APEX_F32) {
        *reinterpret_cast<float4 *>(static_cast<float *>(out) + idx) = make_float4(a, b, c, d);
    } else {
        uint2 v = make_uint2(pack2<DT>(a, b), pack2<DT>(c, d));
        *reinterpret_cast<uint2 *>(static_cast<uint16_t *>(out) + idx) = v;
    }
}

// Final output store: the same 4 values to every destination (n_out <= 8), at
// row b, head (out_head_offset + head).  With peer-mapped destinations (e.g.
// torch symmetric memory over NVLink) this is the all-gather of head-sharded
// outputs fused into the epilogue.
template <int DT>
__device__ __forceinline__ void store_out(const DecodeParams &p, int b, int head, int d4, float a, float bb, float c,
                                          float d) {
    const size_t o = (size_t)b * p.out_row_stride + (size_t)(p.out_head_offset + head) * p.out_head_stride + d4;
#pragma unroll 1
    for (int i = 0; i < p.n_out; ++i) store4<DT>(p.out[i], o, a, bb, c, d);
}

// Completion signal.  Called by every thread of every CTA after
// its last output store: one thread per CTA makes the CTA's stores (local or peer-mapped)
// visible system-wide and counts the CTA; the last CTA of the grid writes signal_value
// into every destination's signal slot with a system-scope release, then re-arms the
// counter.  A reader that acquires the flag (apex_signal_wait) sees all the rows.
__device__ __forceinline__ void signal_done(const DecodeParams &p) {
    if (p.signals[0] == nullptr) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("fence.acq_rel.sys;" ::: "memory");
        if (atomicAdd(p.sig_counter, 1) == (int)gridDim.x - 1) {
            *p.sig_counter = 0;
            asm volatile("fence.acq_rel.sys;" ::: "memory");
            for (int i = 0; i < p.n_out; ++i)
                asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p.signals[i] + p.signal_slot),
                             "r"(p.signal_value)
                             : "memory");
        }
    }
}

// this step's merge list (packed upload: right after the work items, offset in the header)
__device__ __forceinline__ const MergeItem *merges_of(const DecodeParams &p) {
    return reinterpret_cast<const MergeItem *>(reinterpret_cast<const uint8_t *>(p.hdr) + p.hdr->o_merges);
}

// ------------------------------------------------------------------ fused append
// The new token's K and V rows (row b of k_new / v_new, kv head g) as 16-byte
// chunks: i in [0, 2*CPR): tensor i / CPR (0 = K, 1 = V), chunk cc = i % CPR of
// the D-vector (segment cc / 8, 16-B column cc % 8 inside the 128-B segment).
template <int ES> struct NewRow {
    static constexpr int CPR = kHeadDim * ES / 16;   // 16-B chunks per D-vector
    __device__ __forceinline__ static uint4 load(const DecodeParams &p, int b, int g, int i) {
        const uint8_t *src = static_cast<const uint8_t *>(i < CPR ? p.k_new : p.v_new);
        return __ldg(reinterpret_cast<const uint4 *>(src + ((size_t)b * p.num_kv_heads + g) * kHeadDim * ES) +
                     (i % CPR));
    }
    // producer: the row into the pool (layout [blocks][Hkv][2][16][D])
    __device__ __forceinline__ static void to_pool(const DecodeParams &p, int b, int g, int phys, int t, int lane) {
        for (int i = lane; i < 2 * CPR; i += 32) {
            uint8_t *dst = static_cast<uint8_t *>(p.kv_pool) +
                           ((((size_t)phys * p.num_kv_heads + g) * 2 + i / CPR) * kTileRows + t) * kHeadDim * ES;
            reinterpret_cast<uint4 *>(dst)[i % CPR] = load(p, b, g, i);
        }
    }
    // consumer: the row into the 128-B-swizzled smem tile ([segment][32 rows][128 B])
    // over whatever the bulk copy brought for it, before the tile is used
    __device__ __forceinline__ static void to_tile(const DecodeParams &p, int b, int g, uint32_t kt, int t, int lane) {
        for (int i = lane; i < 2 * CPR; i += 32) {
            const uint4 v = load(p, b, g, i);
            const int cc = i % CPR, sg = cc / 8, c = cc % 8, row = (i / CPR) * kTileRows + t;
            const uint32_t a = kt + sg * kSegStride + row * 128 + ((c ^ (row & 7)) << 4);
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                         : "memory");
        }
        // generic-proxy writes to a slot the bulk-copy (async) proxy will refill later
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
    }
};

// ------------------------------------------------------------------ consumers
// CUDA-core consumer for g == 1 (fp32 or 16-bit).  q.K: lane t (0..15) owns token
// t, half hh = lane/16 owns dims hh*64..hh*64+63.  P.V: lane owns 8 (16-bit) or
// 4 (fp32) dims; 16-bit lanes split even/odd tokens by half-warp.
template <int DT> struct SimtConsumer {
    static constexpr bool F32 = DT == APEX_F32;
    float qv[64];               // q * scale*log2e, dims hh*64 ..
    float o[8];                 // 16-bit: 8 dims; fp32: 4 dims (o[0..3])
    float m, l;                 // l: per-lane partial of sum p (lanes 0..15 distinct)

    __device__ __forceinline__ void begin(const uint8_t *qg, const DecodeParams &p, int lane) {
        const int hh = lane >> 4;
        const size_t base = (size_t)hh * 64;
        if constexpr (F32) {
            const float4 *src = reinterpret_cast<const float4 *>(reinterpret_cast<const float *>(qg) + base);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                float4 v = LDQ(src + i);
                qv[4 * i] = v.x * p.scale_log2;
                qv[4 * i + 1] = v.y * p.scale_log2;
                qv[4 * i + 2] = v.z * p.scale_log2;
                qv[4 * i + 3] = v.w * p.scale_log2;
            }
        } else {
            const uint4 *src = reinterpret_cast<const uint4 *>(reinterpret_cast<const uint16_t *>(qg) + base);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                uint4 v = LDQ(src + i);
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    float2 f = unpack2<DT>(w[j]);
                    qv[8 * i + 2 * j] = f.x * p.scale_log2;
                    qv[8 * i + 2 * j + 1] = f.y * p.scale_log2;
                }
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = 0.f;
        m = -INFINITY;
        l = 0.f;
    }

    template <typename Release>
    __device__ __forceinline__ void tile(uint32_t kt, uint32_t vt, int valid, float, int lane, Release release) {
        const int t = lane & 15, hh = lane >> 4, t7 = t & 7;
        // ---- s_t (log2 units): lane t, dims of half hh
        float acc = 0.f;
        if constexpr (F32) {
            // four independent FMA chains (16 deep instead of 64): in the latency regime a
            // warp usually holds one tile, so the dependent-FMA latency is on the critical path
            float a4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int sg = 0; sg < 2; ++sg) {
                const uint32_t rowa = kt + (uint32_t)((2 * hh + sg) * kSegStride + t * 128);
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    uint4 k4 = lds128(rowa + ((c ^ t7) << 4));
                    const float *qq = qv + sg * 32 + c * 4;
                    a4[0] = fmaf(qq[0], __uint_as_float(k4.x), a4[0]);
                    a4[1] = fmaf(qq[1], __uint_as_float(k4.y), a4[1]);
                    a4[2] = fmaf(qq[2], __uint_as_float(k4.z), a4[2]);
                    a4[3] = fmaf(qq[3], __uint_as_float(k4.w), a4[3]);
                }
            }
            acc = (a4[0] + a4[1]) + (a4[2] + a4[3]);
        } else {
            const uint32_t rowa = kt + (uint32_t)(hh * kSegStride + t * 128);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                uint4 k4 = lds128(rowa + ((c ^ t7) << 4));
                const uint32_t w[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    float2 f = unpack2<DT>(w[j]);
                    acc = fmaf(qv[c * 8 + 2 * j], f.x, acc);
                    acc = fmaf(qv[c * 8 + 2 * j + 1], f.y, acc);
                }
            }
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, 16);
        const float x = t < valid ? acc : -INFINITY;
        float mx = x;
#pragma unroll
        for (int w = 1; w < 16; w <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, w));
        const float m_new = fmaxf(m, mx);
        const float alpha = ex2_diff(m, m_new);
        m = m_new;
        const float pt = ex2_diff(x, m_new);
        l = l * alpha + pt;
        if (__any_sync(0xffffffffu, alpha != 1.f)) {   // bit-identical skip when the max did not move
#pragma unroll
            for (int i = 0; i < 8; ++i) o[i] *= alpha;
        }
        // ---- O += p_r V_r over lane-owned dims
        if constexpr (F32) {
            // even rows accumulate into o[0..3], odd rows into o[4..7] (two chains of 8; the
            // halves are added in finish())
            const int sg = lane >> 3, c = lane & 7;
#pragma unroll
            for (int r = 0; r < kTileRows; ++r) {
                const float pr = __shfl_sync(0xffffffffu, pt, r);
                if (r < valid) {
                    uint4 v4 = lds128(vt + (uint32_t)(sg * kSegStride + r * 128) + ((c ^ (r & 7)) << 4));
                    float *oo = o + 4 * (r & 1);
                    oo[0] = fmaf(pr, __uint_as_float(v4.x), oo[0]);
                    oo[1] = fmaf(pr, __uint_as_float(v4.y), oo[1]);
                    oo[2] = fmaf(pr, __uint_as_float(v4.z), oo[2]);
                    oo[3] = fmaf(pr, __uint_as_float(v4.w), oo[3]);
                }
            }
        } else {
            const int sg = (lane & 15) >> 3, c = lane & 7;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int r = 2 * i + hh;
                const float pr = __shfl_sync(0xffffffffu, pt, r);
                if (r < valid) {
                    uint4 v4 = lds128(vt + (uint32_t)(sg * kSegStride + r * 128) + ((c ^ (r & 7)) << 4));
                    const uint32_t w[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        float2 f = unpack2<DT>(w[j]);
                        o[2 * j] = fmaf(pr, f.x, o[2 * j]);
                        o[2 * j + 1] = fmaf(pr, f.y, o[2 * j + 1]);
                    }
                }
            }
        }
        release();
    }

    __device__ __forceinline__ void finish(float *cb_o, float *cb_m, float *cb_l, int wc, int lane) {
#pragma unroll
        for (int w = 1; w < 16; w <<= 1) l += __shfl_xor_sync(0xffffffffu, l, w);
        float *dst = cb_o + (size_t)wc * kHeadDim;
        if constexpr (F32) {
            const int sg = lane >> 3, c = lane & 7;
            *reinterpret_cast<float4 *>(dst + sg * 32 + c * 4) =
                make_float4(o[0] + o[4], o[1] + o[5], o[2] + o[6], o[3] + o[7]);
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) o[i] += __shfl_xor_sync(0xffffffffu, o[i], 16);
            if (lane < 16) {
                const int sg = lane >> 3, c = lane & 7;
                *reinterpret_cast<float4 *>(dst + sg * 64 + c * 8) = make_float4(o[0], o[1], o[2], o[3]);
                *reinterpret_cast<float4 *>(dst + sg * 64 + c * 8 + 4) = make_float4(o[4], o[5], o[6], o[7]);
            }
        }
        if (lane == 0) {
            cb_m[wc] = m;
            cb_l[wc] = l;
        }
    }
};

// Transposed tensor-core consumer for GQA (g >= 2, 16-bit): the q-group is the
// N = 8 side of mma.m16n8k16 instead of padded M = 16 rows, so a 16-token tile
// costs 16 HMMA instead of 48 and the O accumulators halve (32 floats/thread):
//   S^T (16 tok x 8 heads) = K (16 tok x 16 d, A, ldmatrix) * Q^T (B, registers), 8 k-steps
//   O^T (128 d x 8 heads) += V^T (A: ldmatrix.trans of the V rows) * P^T (B)
// P^T's B fragments come from the S^T accumulators by movmatrix.trans (two 8x8
// b16 transposes), the per-head softmax statistics reduce over the 8 lanes
// holding one head column.  Heads >= G have zero q (finite, ignored).
__device__ __forceinline__ uint32_t movmatrix_trans(uint32_t a) {
    uint32_t d;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
    return d;
}
template <int DT>
__device__ __forceinline__ void mma_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
    if constexpr (DT == APEX_BF16)
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    else
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int DT, int G> struct MmaConsumerT {
    uint32_t qb[8][2];          // B fragments of Q^T per k-step: q[h = lane/4][d pairs], zero for h >= G
    float o[8][4];              // O^T accumulators, m-tile md covers dims md*16 .. md*16+15
    float m[2], l[2];           // per head column (lane%4)*2 + j: running max (log2) and partial sum

    __device__ __forceinline__ void begin(const uint8_t *qg, const DecodeParams &, int lane) {
        const int h = lane >> 2, tid = lane & 3;
        const uint32_t *qrow = reinterpret_cast<const uint32_t *>(qg + (size_t)h * kHeadDim * 2);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            qb[kk][0] = h < G ? LDQ(qrow + kk * 8 + tid) : 0u;
            qb[kk][1] = h < G ? LDQ(qrow + kk * 8 + 4 + tid) : 0u;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
        m[0] = m[1] = -INFINITY;
        l[0] = l[1] = 0.f;
    }

    template <typename Release>
    __device__ __forceinline__ void tile(uint32_t kt, uint32_t vt, int valid, float scale_log2, int lane,
                                         Release release) {
        const int tid = lane & 3, t8 = lane >> 2;
        // ---- S^T = K Q^T (16 tokens x 8 heads), 8 k-steps over d
        float sacc[4] = {0.f, 0.f, 0.f, 0.f};
        {
            const int r = lane & 15;                       // K row (token) this lane addresses
            const uint32_t k_lane = kt + (uint32_t)(r * 128);
            const int cx = (lane >> 4) ^ (r & 7);          // chunk kk*2 + (lane >> 4), swizzled
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                uint32_t a0, a1, a2, a3;
                ldsm_x4(k_lane + (kk >> 2) * kSegStride + ((((kk & 3) * 2) ^ cx) << 4), a0, a1, a2, a3);
                mma_16816<DT>(sacc, a0, a1, a2, a3, qb[kk][0], qb[kk][1]);
            }
        }
        // ---- online softmax per head column; rows t8 (c0, c1) and t8 + 8 (c2, c3)
        const bool v0 = t8 < valid, v1 = t8 + 8 < valid;
        float x[4];
        x[0] = v0 ? sacc[0] * scale_log2 : -INFINITY;     // (t8,   head 2tid)
        x[1] = v0 ? sacc[1] * scale_log2 : -INFINITY;     // (t8,   head 2tid+1)
        x[2] = v1 ? sacc[2] * scale_log2 : -INFINITY;     // (t8+8, head 2tid)
        x[3] = v1 ? sacc[3] * scale_log2 : -INFINITY;     // (t8+8, head 2tid+1)
        float mx0 = fmaxf(x[0], x[2]), mx1 = fmaxf(x[1], x[3]);
#pragma unroll
        for (int o_ = 4; o_ < 32; o_ <<= 1) {
            mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o_));
            mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o_));
        }
        const float mn0 = fmaxf(m[0], mx0), mn1 = fmaxf(m[1], mx1);
        const float al0 = ex2_diff(m[0], mn0), al1 = ex2_diff(m[1], mn1);
        m[0] = mn0;
        m[1] = mn1;
        const uint32_t p01 = pack2<DT>(ex2_diff(x[0], mn0), ex2_diff(x[1], mn1));   // P^T rows t8
        const uint32_t p23 = pack2<DT>(ex2_diff(x[2], mn0), ex2_diff(x[3], mn1));   // P^T rows t8 + 8
        // l accumulates the same (rounded) p that feeds the P.V product
        const float2 f01 = unpack2<DT>(p01), f23 = unpack2<DT>(p23);
        l[0] = l[0] * al0 + (f01.x + f23.x);
        l[1] = l[1] * al1 + (f01.y + f23.y);
        // rescale only when some head's running max moved (alpha == 1 exactly otherwise,
        // so skipping is bit-identical; after the first tiles it rarely moves)
        if (__any_sync(0xffffffffu, al0 != 1.f || al1 != 1.f)) {
#pragma unroll
            for (int md = 0; md < 8; ++md) {
                o[md][0] *= al0;
                o[md][1] *= al1;
                o[md][2] *= al0;
                o[md][3] *= al1;
            }
        }
        const uint32_t b0 = movmatrix_trans(p01), b1 = movmatrix_trans(p23);   // P^T as B (k = tokens)
        // ---- O^T += V^T P^T: V^T fragments by ldmatrix.trans; invalid tokens' V zeroed (NaN-safe)
        uint32_t mlo = 0xffffffffu, mhi = 0xffffffffu;
        if (valid < kTileRows) {
            mlo = (tid * 2 < valid ? 0x0000ffffu : 0u) | (tid * 2 + 1 < valid ? 0xffff0000u : 0u);
            mhi = (8 + tid * 2 < valid ? 0x0000ffffu : 0u) | (8 + tid * 2 + 1 < valid ? 0xffff0000u : 0u);
        }
        {
            const int r = (lane & 7) + (lane >> 4) * 8;    // V row (token) this lane addresses
            // 16-B column of m-tile md: ((md % 4) * 2 + b) ^ (r & 7) = ((md % 4) * 2) ^ cx
            const uint32_t v_lane = vt + (uint32_t)(r * 128);
            const int cx = ((lane >> 3) & 1) ^ (r & 7);
            if (valid == kTileRows) {                     // full tile: no masking (uniform branch)
#pragma unroll
                for (int md = 0; md < 8; ++md) {
                    uint32_t a0, a1, a2, a3;
                    ldsm_x4_t(v_lane + (md >> 2) * kSegStride + ((((md & 3) * 2) ^ cx) << 4), a0, a1, a2, a3);
                    mma_16816<DT>(o[md], a0, a1, a2, a3, b0, b1);
                }
            } else {
#pragma unroll
                for (int md = 0; md < 8; ++md) {
                    uint32_t a0, a1, a2, a3;
                    ldsm_x4_t(v_lane + (md >> 2) * kSegStride + ((((md & 3) * 2) ^ cx) << 4), a0, a1, a2, a3);
                    mma_16816<DT>(o[md], a0 & mlo, a1 & mlo, a2 & mhi, a3 & mhi, b0, b1);
                }
            }
        }
        release();
    }

    __device__ __forceinline__ void finish(float *cb_o, float *cb_m, float *cb_l, int wc, int lane) {
        const int tid = lane & 3, t8 = lane >> 2;
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int o_ = 4; o_ < 32; o_ <<= 1) l[j] += __shfl_xor_sync(0xffffffffu, l[j], o_);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int h = tid * 2 + j;
            if (h < G) {
                float *dst = cb_o + ((size_t)wc * G + h) * kHeadDim;
#pragma unroll
                for (int md = 0; md < 8; ++md) {
                    dst[md * 16 + t8] = o[md][j];
                    dst[md * 16 + t8 + 8] = o[md][2 + j];
                }
                if (t8 == 0) {
                    cb_m[wc * G + h] = m[j];
                    cb_l[wc * G + h] = l[j];
                }
            }
        }
    }
};

template <int DT, int G, bool FUSE> struct ConsumerSel { using T = MmaConsumerT<DT, G>; };
// MHA (g = 1): fp32 on CUDA cores.  16-bit: the transposed tensor-core path with one
// live head column (16 HMMA per tile instead of ~260 FMA/unpack instructions per lane):
// faster per tile in the latency regime (fp16 batch 8 x 1K: 43 -> 40 us) and, by
// issuing half the instructions, cooler in the bandwidth regime -- C2 sustained over
// 60 steps under sw_power_cap: 1.51 -> 1.58 GHz, 3,134 -> 3,166 tokens/s (+1.0%,
// same box, 3 rounds); isolated calls 603.0 -> 601.2 us.
template <int DT, bool FUSE> struct ConsumerSel<DT, 1, FUSE> {
    using T = typename std::conditional<DT != APEX_F32, MmaConsumerT<DT, 1>, SimtConsumer<DT>>::type;
};

// log-sum-exp merge of one split (b, g) pair, partials combined in split order:
// M = max m_i, out = sum 2^(m_i-M) O_i / sum 2^(m_i-M) l_i.  Partials written by
// other CTAs are read through L2 (ld.global.cg).
//
// One pass with a running max: thread (output float4 o, part group gr) folds
// parts i = gr, gr + ngr, ... into (M, den, acc) with acc <- acc 2^(M-M') +
// 2^(m_i-M') O_i.  The loads of all parts are independent of the running state,
// so the unrolled loop can keep several parts in flight per thread (inside the
// decode kernel, at its 168-register cap, ptxas serialises part of them: a 37-way
// merge there measures 10-20 dependent L2 round trips, ~3.5 us; batched, staged
// and warp-per-row variants were no faster -- profiles/r02_merge_ab.txt).
// Part groups (ngr = nt / (G * 32) > 1 when the pair has fewer float4 outputs than
// the nt = 128 participating threads) are combined through `red`/`redml` in fixed
// group order.  `sync` is a barrier over the nt participating threads.
template <int DT, int G, typename Sync>
__device__ __forceinline__ void merge_pair(const DecodeParams &p, const MergeItem mg, int t, int nt, float4 *red,
                                           float2 *redml, int red_cap, Sync sync) {
    const int np = mg.nparts;
    constexpr int NOUT = G * kHeadDim / 4;                    // float4 outputs of the pair
    const float2 *ml = reinterpret_cast<const float2 *>(p.part_ml) + (size_t)mg.part0 * G;
    const int ngr = red ? max(1, min(nt, red_cap) / NOUT) : 1;   // part groups (1 when NOUT >= nt)
    for (int idx = t; idx < NOUT * ngr; idx += nt) {
        const int o = idx % NOUT, gr = idx / NOUT;
        const int row = o / (kHeadDim / 4), d4 = (o % (kHeadDim / 4)) * 4;
        const float *po = p.part_o + ((size_t)mg.part0 * G + row) * kHeadDim + d4;
        float M = -INFINITY, den = 0.f, a = 0.f, b = 0.f, c = 0.f, d = 0.f;
#pragma unroll kMergeUnroll
        for (int i = gr; i < np; i += ngr) {
            const float2 mi = __ldcg(ml + (size_t)i * G + row);
            const float4 v = __ldcg(reinterpret_cast<const float4 *>(po + (size_t)i * G * kHeadDim));
            const float Mn = fmaxf(M, mi.x);
            const float al = ex2_diff(M, Mn), e = ex2_diff(mi.x, Mn);
            den = fmaf(den, al, e * mi.y);
            a = fmaf(a, al, e * v.x);
            b = fmaf(b, al, e * v.y);
            c = fmaf(c, al, e * v.z);
            d = fmaf(d, al, e * v.w);
            M = Mn;
        }
        if (ngr == 1) {
            store_out<DT>(p, mg.b, mg.g * G + row, d4, a / den, b / den, c / den, d / den);
        } else {
            red[gr * NOUT + o] = make_float4(a, b, c, d);
            redml[gr * NOUT + o] = make_float2(M, den);
        }
    }
    if (ngr > 1) {
        sync();
        for (int o = t; o < NOUT; o += nt) {
            const int row = o / (kHeadDim / 4), d4 = (o % (kHeadDim / 4)) * 4;
            float M = -INFINITY;
            for (int gr = 0; gr < ngr; ++gr) M = fmaxf(M, redml[gr * NOUT + o].x);
            float den = 0.f, a = 0.f, b = 0.f, c = 0.f, d = 0.f;
            for (int gr = 0; gr < ngr; ++gr) {
                const float2 mlg = redml[gr * NOUT + o];
                const float e = ex2_diff(mlg.x, M);
                const float4 v = red[gr * NOUT + o];
                den = fmaf(e, mlg.y, den);
                a = fmaf(e, v.x, a);
                b = fmaf(e, v.y, b);
                c = fmaf(e, v.z, c);
                d = fmaf(e, v.w, d);
            }
            store_out<DT>(p, mg.b, mg.g * G + row, d4, a / den, b / den, c / den, d / den);
        }
        sync();                                                // red reusable for the next pair
    }
}

// ------------------------------------------------------------------ decode kernel
template <int DT, int G, bool FUSE, bool AP>
__global__ void __launch_bounds__(NTHREADS, CTAS_PER_SM)
    apex_decode_kernel(const __grid_constant__ CUtensorMap tmkv,
                       const DecodeParams p) {
    using C = Cfg<DT, G, FUSE>;
    using S = C;
    constexpr int STAGES = C::STAGES, TILE = C::TILE;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + S::TILES);
    ItemSlot *ring = reinterpret_cast<ItemSlot *>(smem + S::TILES + S::BARS);
    float *cb_o = reinterpret_cast<float *>(smem + S::TILES + S::BARS + S::RING);
    float *cb_m = cb_o + NC * G * kHeadDim;
    float *cb_l = cb_m + NC * G;
    volatile int *merge_flag = reinterpret_cast<volatile int *>(cb_l + NC * G);
    float4 *mred = reinterpret_cast<float4 *>(smem + S::TILES + S::BARS + S::RING + S::CB_O + S::CB_ML);
    float2 *mredml = reinterpret_cast<float2 *>(mred + NC * 32);
    const uint32_t tiles_u = smem_u32(smem);
    const uint32_t full0 = smem_u32(bars), empty0 = full0 + 8 * STAGES;
    const uint32_t ifull0 = empty0 + 8 * STAGES, iempty0 = ifull0 + 8 * IR;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) TRACE(0);
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(full0 + 8 * i, 1);
            mbar_init(empty0 + 8 * i, 1);
        }
        for (int i = 0; i < IR; ++i) {
            mbar_init(ifull0 + 8 * i, 1);
            mbar_init(iempty0 + 8 * i, NC);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmkv)) : "memory");
    }
    __syncthreads();
    // PDL: everything above overlapped the previous kernel; from here on we read
    // its results (pools, block table, lengths).  Dependents (the merge kernel)
    // may be scheduled now; they wait on their own griddepcontrol.wait.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0) TRACE(1);

    if (warp == 0) {
        // ================= producer: work queue + block table + TMA =================
        // Measured alternatives: running the next item's control
        // loads ahead in this warp (7-13% slower: the dependent round trips then stall
        // the TMA stream mid-item), and a separate scheduler warp feeding item, q and
        // block ids through shared memory (no faster at the default split, +1 warp).
        const int n_items = p.hdr->n_items;    // this step's work-list length (device header)
        int s_next = __ldg(p.cta_begin + blockIdx.x);
        const int s_end = __ldg(p.cta_begin + blockIdx.x + 1), q_base = __ldg(p.cta_begin + gridDim.x);
        // speculative load of item blockIdx.x (the first item of CTA i is item i unless the
        // plan has stream-K ranges): issued together with the header loads, one round
        // trip earlier than a load that waits for cta_begin (the list has >= grid slots)
        const WorkItem spec = p.items[blockIdx.x].it;
        const int spec_ids = lane < kInlineIds ? p.items[blockIdx.x].ids[lane] : 0;
        // lane w < NC: consumer warp w's sub-ring as (next slot, completed passes), kept
        // incrementally -- no division by SW and no run-time warp selection on the per-tile
        // path (measured: C5 +1.9%, C3 +1.2% sustained against m % SW, m / SW with one lane
        // issuing for all warps; issuing from NC lanes in parallel: C2 +1.1%, others equal)
        int32_t rs = 0, ru = 0;
        const int hkv = p.num_kv_heads;
        const bool one_op = p.tma_segs == 1;
        for (int k = 0;; ++k) {
            int idx;
            if (s_next < s_end) {
                idx = s_next++;
            } else {
                if (lane == 0) idx = q_base + atomicAdd(p.counters, 1);
                idx = __shfl_sync(0xffffffffu, idx, 0);
            }
            const int slot = k % IR, use = k / IR;
            if (lane == 0 && use > 0) mbar_wait(iempty0 + 8 * slot, (use - 1) & 1);
            __syncwarp();
            if (idx >= n_items) {
                if (lane == 0) {
                    ring[slot].it.nblk = 0;   // sentinel: no more items
                    mbar_arrive(ifull0 + 8 * slot);
                }
                break;
            }
            const bool use_spec = APEX_SPEC_ITEM && k == 0 && idx == (int)blockIdx.x;
            const WorkItem it = use_spec ? spec : p.items[idx].it;
            // physical ids of the item's first kInlineIds blocks, loaded with the item: the
            // first TMAs do not wait for the dependent block-table load below
            const int inl = use_spec ? spec_ids : (lane < kInlineIds ? p.items[idx].ids[lane] : 0);
            if (lane == 0) {
                ring[slot].it = it;
                mbar_arrive(ifull0 + 8 * slot);
                if (k == 0) TRACE(2);
            }
            const int32_t *bt = p.block_table + (size_t)it.seq * p.max_blocks_per_seq + it.blk0;
            // lane w < NC feeds consumer warp w's sub-ring: it issues tiles j = w, w + NC, ...
            // of the item, in order, with its own (slot, pass) counters, so the NC sub-rings
            // are refilled in parallel and the per-tile path is one shuffle + one TMA
            const int tl = AP ? (it.len - 1) / kTileRows - it.blk0 : -1;   // fused append: block of the new row
            for (int j0 = 0; j0 < it.nblk; j0 += 32) {
                const int my = j0 + lane < it.nblk ? (j0 + lane < kInlineIds ? inl : __ldg(bt + j0 + lane)) : 0;
                const int cnt = min(32, it.nblk - j0);
#ifdef APEX_TRACE
                if (k == 0 && j0 == 0) {
                    __shfl_sync(0xffffffffu, my, 0);
                    if (lane == 0) TRACE(3);
                }
#endif
                if (AP && tl >= j0 && tl < j0 + cnt)                        // warp-uniform
                    NewRow<C::ES>::to_pool(p, it.b, it.g, __shfl_sync(0xffffffffu, my, tl - j0),
                                           (it.len - 1) % kTileRows, lane);
                for (int jj = 0; jj < cnt; jj += NC) {
                    const int phys = __shfl_sync(0xffffffffu, my, (jj + lane) & 31);
                    if (lane < NC && jj + lane < cnt) {
                        const int s = lane * C::SW + rs;
                        if (ru > 0) mbar_wait(empty0 + 8 * s, (ru - 1) & 1);
                        const uint32_t bar = full0 + 8 * s;
                        mbar_expect_tx(bar, 2 * TILE);
                        const int row = (phys * hkv + it.g) * 2 * kTileRows;   // K row 0 of the tile
                        const uint32_t dk = tiles_u + s * 2 * TILE;
                        if (one_op) {
                            tma_load_3d(dk, &tmkv, bar, 0, row, 0);     // K and V of the tile, 1 op
                        } else {
                            for (int sg = 0; sg < p.tma_segs; ++sg)
                                tma_load_2d(dk + sg * kSegStride, &tmkv, bar, sg * (128 / C::ES), row);
                        }
                        if (++rs == C::SW) {                            // next slot of this sub-ring
                            rs = 0;
                            ++ru;
                        }
                    }
                }
            }
        }
        // last CTA out resets the queue for the next launch on this layer
        if (lane == 0) {
            TRACE(4);
            __threadfence();
            if (atomicAdd(p.counters + 1, 1) == (int)gridDim.x - 1) {
                atomicExch(p.counters, 0);
                atomicExch(p.counters + 1, 0);
            }
        }
    } else {
        // ================= consumers =================
        const int wc = warp - 1;
        typename ConsumerSel<DT, G, FUSE>::T st;
        int32_t cs = 0;                       // this warp's sub-ring position: slot, phase parity
        uint32_t cph = 0;
        for (int k = 0;; ++k) {
            const int slot = k % IR, use = k / IR;
            mbar_wait(ifull0 + 8 * slot, use & 1);
            const WorkItem it = ring[slot].it;
            if (it.nblk == 0) break;
            // the pair's merge record, loaded now so that the arrival test and the fused merge
            // at the item's end do not start with a dependent (after an L2 flush: DRAM) load
            MergeItem mgi{};
            if (FUSE && it.part >= 0) mgi = merges_of(p)[it.mg];
            st.begin(static_cast<const uint8_t *>(p.q) +
                         ((size_t)it.b * p.num_q_heads + (size_t)it.g * G) * kHeadDim * C::ES, p, lane);
            __syncwarp();
            if (lane == 0) mbar_arrive(iempty0 + 8 * slot);   // item and q slot read
            for (int j = wc; j < it.nblk; j += NC) {
                const int s = wc * C::SW + cs;
                mbar_wait(full0 + 8 * s, cph);
                if (++cs == C::SW) {                     // next slot of this warp's sub-ring
                    cs = 0;
                    cph ^= 1u;
                }
#ifdef APEX_TRACE
                if (k == 0 && j == 0 && lane == 0 && wc == 0) TRACE(5);
#endif
                const int valid = min(kTileRows, it.len - (it.blk0 + j) * kTileRows);
                const uint32_t kt = tiles_u + s * 2 * TILE;
                if (AP && it.blk0 + j == (it.len - 1) / kTileRows)   // fused append: patch the new row
                    NewRow<C::ES>::to_tile(p, it.b, it.g, kt, (it.len - 1) % kTileRows, lane);
                st.tile(kt, kt + kVOff, valid, p.scale_log2, lane, [&] {
                    __syncwarp();                                 // every lane's smem reads of the slot are done
                    if (lane == 0) mbar_arrive(empty0 + 8 * s);   // release it to the producer
                });
            }
#ifdef APEX_TRACE
            if (k == 0 && lane == 0 && wc == 0) TRACE(6);
#endif
            st.finish(cb_o, cb_m, cb_l, wc, lane);
            named_bar_sync(1, NC * 32);
#ifdef APEX_TRACE
            if (k == 0 && threadIdx.x == 32) TRACE(7);
#endif
            // ---- merge the NC warp states (fixed order), 4 dims per step
            for (int idx = threadIdx.x - 32; idx < G * kHeadDim / 4; idx += NC * 32) {
                const int row = idx / (kHeadDim / 4), d4 = (idx % (kHeadDim / 4)) * 4;
                float M = -INFINITY;
#pragma unroll
                for (int w = 0; w < NC; ++w) M = fmaxf(M, cb_m[w * G + row]);
                float den = 0.f, a = 0.f, b = 0.f, c = 0.f, d = 0.f;
#pragma unroll
                for (int w = 0; w < NC; ++w) {
                    const float e = ex2_diff(cb_m[w * G + row], M);
                    const float4 v = *reinterpret_cast<const float4 *>(cb_o + ((size_t)w * G + row) * kHeadDim + d4);
                    den = fmaf(e, cb_l[w * G + row], den);
                    a = fmaf(e, v.x, a);
                    b = fmaf(e, v.y, b);
                    c = fmaf(e, v.z, c);
                    d = fmaf(e, v.w, d);
                }
                if (it.part < 0) {
                    store_out<DT>(p, it.b, it.g * G + row, d4, a / den, b / den, c / den, d / den);
                } else {
                    const size_t o = ((size_t)it.part * G + row) * kHeadDim + d4;
                    *reinterpret_cast<float4 *>(p.part_o + o) = make_float4(a, b, c, d);
                    if (d4 == 0) *reinterpret_cast<float2 *>(p.part_ml + ((size_t)it.part * G + row) * 2) = make_float2(M, den);
                }
            }
#ifdef APEX_TRACE
            if (k == 0 && threadIdx.x == 32) TRACE(8);
#endif
            if (FUSE && it.part >= 0) {
                // last-arriving split of this (b, g) pair merges all its partials (fused LSE
                // merge).  Release/acquire through one thread (CUTLASS-semaphore pattern):
                // bar.sync orders the CTA's partial stores before thread 32's gpu-scope
                // acq_rel fence + counter atomic; the last arriver's fence + bar.sync order
                // the other CTAs' partials before every thread's loads (no per-thread
                // sequentially consistent __threadfence).
                named_bar_sync(1, NC * 32);
                if (threadIdx.x == 32) {
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
#ifdef APEX_TRACE
                    if (k == 0) TRACE(13);
#endif
                    const int done = atomicAdd(p.merge_counters + it.mg, 1);
                    const int last = done == mgi.nparts - 1;
                    if (last) {
                        p.merge_counters[it.mg] = 0;            // every split has arrived: re-arm
                        asm volatile("fence.acq_rel.gpu;" ::: "memory");
                    }
                    *merge_flag = last;
                }
                named_bar_sync(1, NC * 32);
#ifdef APEX_TRACE
                if (k == 0 && threadIdx.x == 32) {
                    TRACE(9);
                    TRACE_VAL(14, (unsigned long long)it.mg + 1);
                    TRACE_VAL(15, (unsigned long long)*merge_flag);
                }
#endif
                if (*merge_flag) {
                    merge_pair<DT, G>(p, mgi, threadIdx.x - 32, NC * 32, mred, mredml, NC * 32,
                                      [] { named_bar_sync(1, NC * 32); });
#ifdef APEX_TRACE
                    named_bar_sync(1, NC * 32);
                    if (threadIdx.x == 32) TRACE(10);
#endif
                }
            }
            named_bar_sync(1, NC * 32);
        }
        if (threadIdx.x == 32) TRACE(11);
    }
    // one launch per call (fused merge): this kernel stored every output row.  Otherwise
    // the merge kernel signals; this kernel's rows are flushed by its completion.
    if (FUSE) {
        signal_done(p);
#ifdef APEX_TRACE
        if (threadIdx.x == 0) TRACE(12);
#endif
    } else if (p.signals[0] != nullptr) {
        __syncthreads();   // this CTA's (possibly peer-mapped) rows before the merge kernel's signal
        if (threadIdx.x == 0) asm volatile("fence.acq_rel.sys;" ::: "memory");
    }
}

// log-sum-exp merge of split pairs as its own launch (bandwidth regime): one CTA
// per (b, g) pair, so merging never stalls a decode CTA's TMA stream.
// 128 threads: the bandwidth regime's merges have small fan-in (guided split:
// <= ~20 parts) and many pairs (C3: 1024), so CTA count per wave matters more
// than part groups (512 threads: 13.4 us per C3 layer vs 9.9 us); large fan-in
// occurs only in the latency regime, merged in-kernel.
constexpr int kMergeThreads = 128;
template <int DT, int G>
__global__ void __launch_bounds__(kMergeThreads) apex_merge_kernel(const DecodeParams p) {
    __shared__ float4 red[kMergeThreads];                   // part-group partials (G * 32 * ngr)
    __shared__ float2 redml[kMergeThreads];
    asm volatile("griddepcontrol.wait;" ::: "memory");     // partials of the decode kernel
    const int n = p.hdr->n_merges;                          // fixed grid, grid-stride over this step's pairs
    for (int i = blockIdx.x; i < n; i += gridDim.x)
        merge_pair<DT, G>(p, merges_of(p)[i], threadIdx.x, blockDim.x, red, redml, kMergeThreads,
                          [] { __syncthreads(); });
    signal_done(p);   // runs after the decode grid completed (griddepcontrol.wait): all rows stored
}

template <int DT, int G> cudaError_t prepare() {
    // AP (fused append) is a separate instantiation: its per-tile checks and row
    // copies cost the plain kernel ~8% at C5 sizes when compiled in (measured)
    const void *k[4] = {(const void *)apex_decode_kernel<DT, G, false, false>,
                        (const void *)apex_decode_kernel<DT, G, false, true>,
                        (const void *)apex_decode_kernel<DT, G, true, false>,
                        (const void *)apex_decode_kernel<DT, G, true, true>};
    const int sm[4] = {Cfg<DT, G, false>::TOTAL, Cfg<DT, G, false>::TOTAL, Cfg<DT, G>::TOTAL, Cfg<DT, G>::TOTAL};
    for (int i = 0; i < 4; ++i) {
        cudaError_t e = cudaFuncSetAttribute(k[i], cudaFuncAttributeMaxDynamicSharedMemorySize, sm[i]);
        if (e != cudaSuccess) return e;
    }
    // load the merge kernel now as well (see append_prepare)
    cudaFuncAttributes a;
    return cudaFuncGetAttributes(&a, apex_merge_kernel<DT, G>);
}

// Decode and merge kernels are launched with programmatic dependent launch:
// their prologue (barrier init, descriptor prefetch) overlaps the tail of the
// previous kernel on the stream, and griddepcontrol.wait orders every read of
// the previous kernel's results.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), int grid, int block, int smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <int DT, int G>
cudaError_t launch(const TmaMap &tm, const DecodeParams &p, int grid, cudaStream_t s) {
    if (grid > 0) {
        const bool ap = p.k_new != nullptr;
        cudaError_t e;
        if (p.fuse_merge)
            e = ap ? launch_pdl(apex_decode_kernel<DT, G, true, true>, grid, NTHREADS, Cfg<DT, G>::TOTAL, s, tm.kv, p)
                   : launch_pdl(apex_decode_kernel<DT, G, true, false>, grid, NTHREADS, Cfg<DT, G>::TOTAL, s, tm.kv, p);
        else
            e = ap ? launch_pdl(apex_decode_kernel<DT, G, false, true>, grid, NTHREADS, Cfg<DT, G, false>::TOTAL, s,
                                tm.kv, p)
                   : launch_pdl(apex_decode_kernel<DT, G, false, false>, grid, NTHREADS, Cfg<DT, G, false>::TOTAL, s,
                                tm.kv, p);
        if (e != cudaSuccess || p.fuse_merge) return e;
    }
    // launched whenever merges are not fused, even if this step has none (it then
    // exits at once): the launch sequence never depends on the step's plan
    return launch_pdl(apex_merge_kernel<DT, G>, p.merge_grid, kMergeThreads, 0, s, p);
}

}  // namespace

#ifdef APEX_TRACE
extern "C" int apex_debug_trace(unsigned long long *host, int n) {
    cudaDeviceSynchronize();
    return (int)cudaMemcpyFromSymbol(host, g_apex_trace, sizeof(unsigned long long) * 16 * (size_t)n);
}
extern "C" int apex_debug_trace_clear(void) {
    static unsigned long long zero[1024][16];
    return (int)cudaMemcpyToSymbol(g_apex_trace, zero, sizeof zero);
}
#endif

bool decode_supported(apex_dtype dt, int group) {
    if (dt == APEX_F32) return group == 1;
    return group == 1 || group == 2 || group == 4 || group == 8;
}

int decode_grid_ctas(apex_dtype, int, int sm_count) { return CTAS_PER_SM * sm_count; }

cudaError_t decode_prepare(apex_dtype dt, int group) {
    if (!decode_supported(dt, group)) return cudaErrorInvalidValue;
    switch (dt) {
    case APEX_F32: return prepare<APEX_F32, 1>();
    case APEX_F16:
        switch (group) {
        case 1: return prepare<APEX_F16, 1>();
        case 2: return prepare<APEX_F16, 2>();
        case 4: return prepare<APEX_F16, 4>();
        default: return prepare<APEX_F16, 8>();
        }
    default:
        switch (group) {
        case 2: return prepare<APEX_BF16, 2>();
        case 4: return prepare<APEX_BF16, 4>();
        default: return prepare<APEX_BF16, 8>();
        }
    }
}

cudaError_t launch_decode(apex_dtype dt, int group, const TmaMap &tm, const DecodeParams &p, int grid,
                          cudaStream_t s) {
    if (!decode_supported(dt, group)) return cudaErrorInvalidValue;
#define APEX_LAUNCH_ARGS (tm, p, grid, s)
    switch (dt) {
    case APEX_F32: return launch<APEX_F32, 1> APEX_LAUNCH_ARGS;
    case APEX_F16:
        switch (group) {
        case 1: return launch<APEX_F16, 1> APEX_LAUNCH_ARGS;
        case 2: return launch<APEX_F16, 2> APEX_LAUNCH_ARGS;
        case 4: return launch<APEX_F16, 4> APEX_LAUNCH_ARGS;
        default: return launch<APEX_F16, 8> APEX_LAUNCH_ARGS;
        }
    default:
        switch (group) {
        case 2: return launch<APEX_BF16, 2> APEX_LAUNCH_ARGS;
        case 4: return launch<APEX_BF16, 4> APEX_LAUNCH_ARGS;
        default: return launch<APEX_BF16, 8> APEX_LAUNCH_ARGS;
        }
    }
#undef APEX_LAUNCH_ARGS
}

}  // namespace apex
