// Read-bandwidth ceiling probe for this B200: how fast can
// a kernel only READ HBM?  MEASURED_PEAKS.json's hbm_gbs is a torch copy
// (read + write).  Variants: (a) LDG.128 grid-stride read + xor-reduce,
// (b) TMA bulk copies (cp.async.bulk) of 8 KiB chunks into a shared-memory ring.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/hbm_probe.cu -o /tmp/hbm_probe && /tmp/hbm_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void ldg_read(const uint4 *__restrict__ p, size_t n, uint32_t *sink) {
    uint32_t acc = 0;
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
#pragma unroll 4
    for (; i < n; i += stride) {
        uint4 v = __ldg(p + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) *sink = acc;
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}" ::"r"(bar), "r"(ph) : "memory");
}

template <int STAGES, int CHUNK>
__global__ void __launch_bounds__(32) bulk_read(const uint8_t *p, size_t chunks, uint32_t *sink) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bars[STAGES];
    const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(bars), s0 = (uint32_t)__cvta_generic_to_shared(sm);
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0 + 8 * i));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    if (threadIdx.x != 0) return;
    size_t k = 0;
    uint32_t acc = 0;
    for (size_t c = blockIdx.x; c < chunks; c += gridDim.x, ++k) {
        const int s = k % STAGES;
        if (k >= STAGES) {
            mbar_wait(b0 + 8 * s, ((k / STAGES) - 1) & 1);
            acc ^= sm[s * CHUNK];
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b0 + 8 * s), "r"(CHUNK) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(s0 + s * CHUNK), "l"(p + c * CHUNK), "r"(CHUNK), "r"(b0 + 8 * s) : "memory");
    }
    for (size_t j = (k > STAGES ? k - STAGES : 0); j < k; ++j) mbar_wait(b0 + 8 * (j % STAGES), (j / STAGES) & 1);
    if (acc == 0x12345678u) *sink = acc;
}

int main() {
    const size_t bytes = 16ull << 30;
    uint8_t *buf;
    uint32_t *sink;
    cudaMalloc(&buf, bytes);
    cudaMalloc(&sink, 4);
    cudaMemset(buf, 1, bytes);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 0;
    for (int occ : {4, 8, 16}) {
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(a);
            ldg_read<<<sms * occ, 256>>>((const uint4 *)buf, bytes / 16, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep) best = best > bytes / ms / 1e6 ? best : bytes / ms / 1e6;
        }
        printf("ldg_read  grid=%d x 256: best %.1f GB/s\n", sms * occ, best);
        best = 0;
    }
    auto bulk = [&](auto kern, int st, int ch) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, st * ch);
        for (int occ : {2, 4}) {
            for (int rep = 0; rep < 5; ++rep) {
                cudaEventRecord(a);
                kern<<<sms * occ, 32, st * ch>>>(buf, bytes / ch, sink);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (rep) best = best > bytes / ms / 1e6 ? best : bytes / ms / 1e6;
            }
            printf("bulk_read grid=%d, %d x %d KiB ring: best %.1f GB/s\n", sms * occ, st, ch / 1024, best);
            best = 0;
        }
    };
    // chunk-size sensitivity at ~96 KiB in flight per CTA
    bulk(bulk_read<12, 8192>, 12, 8192);
    bulk(bulk_read<6, 16384>, 6, 16384);
    bulk(bulk_read<3, 32768>, 3, 32768);
    bulk(bulk_read<24, 4096>, 24, 4096);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
