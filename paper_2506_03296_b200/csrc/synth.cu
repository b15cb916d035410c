// Device twin of synth/gen.py (see include/apex_synth.h).  Input generation
// only -- no part of the attention method.  Checked bit-for-bit against the
// host generator by tests/test_generator_gpu.py.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "../../include/apex_synth.h"
#include "apex_internal.h"

namespace {

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint32_t lowbias32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    return x ^ (x >> 16);
}

// key field shifts (must match synth/gen.py)
constexpr int kT = 8, kH = 26, kB = 33, kL = 49, kX = 55;

template <int DT>
__global__ void __launch_bounds__(256) apex_synth_kernel(void *out, int tensor, int layer, const int32_t *row_b,
                                                         const int32_t *row_pos, int64_t n_rows, int n_heads,
                                                         int head_offset, int head_dim, uint64_t seedmix, float amp) {
    // one thread per 8 consecutive dims of one (row, head)
    const int per_vec = head_dim / 8;
    const int64_t n8 = n_rows * n_heads * per_vec;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
        const int d0 = (int)(i % per_vec) * 8;
        const int64_t rh = i / per_vec;
        const int h = (int)(rh % n_heads);
        const int64_t r = rh / n_heads;
        const uint64_t base = ((uint64_t)tensor << kX) | ((uint64_t)layer << kL) | ((uint64_t)row_b[r] << kB) |
                              ((uint64_t)(head_offset + h) << kH) | ((uint64_t)row_pos[r] << kT);
        const uint64_t hrow = splitmix64(base ^ seedmix);
        const uint32_t lo = (uint32_t)hrow, hi = (uint32_t)(hrow >> 32);
        float x[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const uint32_t u = lowbias32(lo + (uint32_t)(d0 + e) * 0x9E3779B9u) ^ hi;
            const int32_t v = (int32_t)(u >> 8) - (1 << 23);
            x[e] = ((float)v * 2.384185791015625e-07f) * amp;   // 2^-22, exact
        }
        const int64_t o = i * 8;
        if constexpr (DT == APEX_F32) {
            float4 *p = reinterpret_cast<float4 *>(static_cast<float *>(out) + o);
            p[0] = make_float4(x[0], x[1], x[2], x[3]);
            p[1] = make_float4(x[4], x[5], x[6], x[7]);
        } else {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if constexpr (DT == APEX_BF16) {
                    __nv_bfloat162 v = __floats2bfloat162_rn(x[2 * e], x[2 * e + 1]);
                    w[e] = *reinterpret_cast<uint32_t *>(&v);
                } else {
                    __half2 v = __floats2half2_rn(x[2 * e], x[2 * e + 1]);
                    w[e] = *reinterpret_cast<uint32_t *>(&v);
                }
            }
            *reinterpret_cast<uint4 *>(static_cast<uint16_t *>(out) + o) = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
}

}  // namespace

extern "C" apex_status apex_synth_rows(void *out, apex_dtype dtype, int32_t tensor, int32_t layer,
                                       const int32_t *row_b, const int32_t *row_pos, int64_t n_rows, int32_t n_heads,
                                       int32_t head_offset, int32_t head_dim, uint64_t seed, float amp,
                                       apex_stream stream) {
    if (n_rows < 0 || n_heads < 1 || head_dim < 8 || head_dim % 8 || tensor < 0 || tensor > 3 || layer < 0 ||
        layer > 63 || head_offset < 0 || head_offset + n_heads > 128 || head_dim > 256)
        return APEX_EINVAL;
    if (n_rows == 0) return APEX_OK;
    if (!out || !row_b || !row_pos || ((uintptr_t)out & 15)) return APEX_EINVAL;
    const uint64_t seedmix = splitmix64(seed);
    const int64_t n8 = n_rows * n_heads * (head_dim / 8);
    int64_t blocks = (n8 + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    cudaStream_t s = (cudaStream_t)stream;
    switch (dtype) {
    case APEX_F32:
        apex_synth_kernel<APEX_F32><<<(int)blocks, 256, 0, s>>>(out, tensor, layer, row_b, row_pos, n_rows, n_heads,
                                                                head_offset, head_dim, seedmix, amp);
        break;
    case APEX_F16:
        apex_synth_kernel<APEX_F16><<<(int)blocks, 256, 0, s>>>(out, tensor, layer, row_b, row_pos, n_rows, n_heads,
                                                                head_offset, head_dim, seedmix, amp);
        break;
    case APEX_BF16:
        apex_synth_kernel<APEX_BF16><<<(int)blocks, 256, 0, s>>>(out, tensor, layer, row_b, row_pos, n_rows, n_heads,
                                                                 head_offset, head_dim, seedmix, amp);
        break;
    default: return APEX_EINVAL;
    }
    return cudaGetLastError() == cudaSuccess ? APEX_OK : APEX_ECUDA;
}
