// Completion signals for the head-sharded output gather fused into the decode
// epilogue (B200 analogue of hiding the attention-output
// transfer, §2.2).  The decode launch of rank r stores its head
// slice into every rank's (symmetric, peer-mapped) output buffer and then posts
// signal_value into slot r of every rank's signal array (decode.cu
// signal_done).  A reader enqueues apex_signal_wait on its own array before
// anything that reads the gathered rows; the post kernel below lets a reader
// hand a buffer back ("consumed") to the writers for the write-after-read guard.
#include "apex_internal.h"

namespace apex {
namespace {

__global__ void apex_signal_wait_kernel(const uint32_t *signals, int n, uint32_t value, uint64_t timeout_ns,
                                        uint32_t *status) {
    // one warp: lane i polls entries i, i+32, ...  (acquire at system scope)
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = threadIdx.x; i < n; i += 32) {
        for (;;) {
            uint32_t v;
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(signals + i) : "memory");
            // wrap-safe "v >= value" on a 32-bit epoch counter
            if ((int32_t)(v - value) >= 0) break;
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > timeout_ns) {
                if (status) atomicExch(status, 1u);
                break;
            }
            __nanosleep(64);
        }
    }
    __syncwarp();
    // order the flag acquisitions before every later kernel's loads of the rows
    if (threadIdx.x == 0) asm volatile("fence.acq_rel.sys;" ::: "memory");
}

struct PostArgs {
    uint32_t *dst[kMaxOut];
};

__global__ void apex_signal_post_kernel(PostArgs a, int n_dst, int slot, uint32_t value) {
    // everything this stream wrote before (earlier kernels) is flushed at kernel
    // boundaries; the release makes it visible to the peers that acquire the flag
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    if (threadIdx.x < n_dst)
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.dst[threadIdx.x] + slot), "r"(value) : "memory");
}

}  // namespace

cudaError_t launch_signal_wait(const uint32_t *signals, int n, uint32_t value, uint64_t timeout_ns, uint32_t *status,
                               cudaStream_t s) {
    apex_signal_wait_kernel<<<1, 32, 0, s>>>(signals, n, value, timeout_ns, status);
    return cudaPeekAtLastError();
}

cudaError_t launch_signal_post(uint32_t *const *dst, int n_dst, int slot, uint32_t value, cudaStream_t s) {
    PostArgs a{};
    for (int i = 0; i < n_dst; ++i) a.dst[i] = dst[i];
    apex_signal_post_kernel<<<1, 32, 0, s>>>(a, n_dst, slot, value);
    return cudaPeekAtLastError();
}

cudaError_t signal_prepare() {
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, apex_signal_wait_kernel);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, apex_signal_post_kernel);
    return e;
}

}  // namespace apex
