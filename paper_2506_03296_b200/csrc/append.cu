// KV append (one K and one V vector per token per layer) and the
// per-step block-table / length delta application (P:156 dynamic KV management).
//
// append: one thread per 16-byte chunk of a (row, head) vector; 128-bit loads
// and stores.  Pool layout [num_blocks][Hkv][2][16][D]: the K rows and then the
// V rows of one (block, head) form one contiguous 8 KiB (16-bit) / 16 KiB (fp32)
// tile that the decode kernel fetches with a single TMA.  Pure bit copy.
#include "apex_internal.h"

namespace apex {
namespace {

__global__ void __launch_bounds__(256) apex_append_kernel(const uint4 *__restrict__ k_new,
                                                          const uint4 *__restrict__ v_new, uint4 *__restrict__ kv_pool,
                                                          const int32_t *slots,
                                                          const StepHeader *__restrict__ hdr, int hkv,
                                                          int chunks_per_vec) {
    const int n_rows = hdr->n_rows;                       // step count from the device header
    if (!slots)                                           // packed upload: slot map after the merge list
        slots = reinterpret_cast<const int32_t *>(reinterpret_cast<const uint8_t *>(hdr) + hdr->o_slots);
    const int64_t per_tensor = (int64_t)n_rows * hkv * chunks_per_vec;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 2 * per_tensor; i += stride) {
        const bool is_v = i >= per_tensor;
        const int64_t j = is_v ? i - per_tensor : i;
        const int c = (int)(j % chunks_per_vec);
        const int64_t rh = j / chunks_per_vec;
        const int h = (int)(rh % hkv);
        const int64_t row = rh / hkv;
        const int32_t slot = __ldg(slots + row);
        const int64_t blk = slot / kBlock, t = slot % kBlock;
        const int64_t dst = (((blk * hkv + h) * 2 + (is_v ? 1 : 0)) * kBlock + t) * chunks_per_vec + c;
        kv_pool[dst] = __ldg((is_v ? v_new : k_new) + j);
    }
}

__global__ void apex_apply_deltas_kernel(const int2 *__restrict__ bt_delta, int n_bt,
                                         const int2 *__restrict__ len_delta, int n_len,
                                         int32_t *__restrict__ block_table, int32_t *__restrict__ seq_lens) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_bt + n_len; i += gridDim.x * blockDim.x) {
        if (i < n_bt) {
            const int2 d = bt_delta[i];
            block_table[d.x] = d.y;
        } else {
            const int2 d = len_delta[i - n_bt];
            seq_lens[d.x] = d.y;
        }
    }
}

// One launch instead of an H2D copy + the delta kernel: the step metadata is read
// straight from the mapped pinned staging buffer (zero-copy over PCIe) into the device
// upload region, and the table / length deltas are applied from the same host copy.
__global__ void apex_upload_kernel(const uint4 *__restrict__ src, uint4 *__restrict__ dst, int n16,
                                   const int2 *__restrict__ bt_delta, int n_bt, const int2 *__restrict__ len_delta,
                                   int n_len, int32_t *__restrict__ block_table, int32_t *__restrict__ seq_lens) {
    const int nth = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n16 + n_bt + n_len; i += nth) {
        if (i < n16) {
            dst[i] = src[i];
        } else if (i < n16 + n_bt) {
            const int2 d = bt_delta[i - n16];
            block_table[d.x] = d.y;
        } else {
            const int2 d = len_delta[i - n16 - n_bt];
            seq_lens[d.x] = d.y;
        }
    }
}

}  // namespace

cudaError_t launch_upload(const void *host_src, void *dev_dst, size_t bytes, const int2 *bt_delta, int n_bt,
                          const int2 *len_delta, int n_len, int32_t *block_table, int32_t *seq_lens, int sm_count,
                          cudaStream_t s) {
    const int n16 = (int)(bytes / 16);
    const int n = n16 + n_bt + n_len;
    const int blocks = (n + 255) / 256 < 2 * sm_count ? (n + 255) / 256 : 2 * sm_count;
    apex_upload_kernel<<<blocks, 256, 0, s>>>(static_cast<const uint4 *>(host_src), static_cast<uint4 *>(dev_dst), n16,
                                               bt_delta, n_bt, len_delta, n_len, block_table, seq_lens);
    return cudaGetLastError();
}

cudaError_t launch_apply_deltas(const int2 *bt_delta, int n_bt, const int2 *len_delta, int n_len,
                                int32_t *block_table, int32_t *seq_lens, cudaStream_t s) {
    const int n = n_bt + n_len;
    if (n == 0) return cudaSuccess;
    const int blocks = (n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024;
    apex_apply_deltas_kernel<<<blocks, 256, 0, s>>>(bt_delta, n_bt, len_delta, n_len, block_table, seq_lens);
    return cudaGetLastError();
}

// Fixed grid (grid-stride over hdr->n_rows) so the launch is step-invariant.
cudaError_t launch_append(apex_dtype dt, const void *k_new, const void *v_new, void *kv_pool,
                          const int32_t *slots, const StepHeader *hdr, int n_kv_heads, int sm_count,
                          cudaStream_t s) {
    const int es = dt == APEX_F32 ? 4 : 2;
    const int cpv = kHeadDim * es / 16;
    apex_append_kernel<<<sm_count * 8, 256, 0, s>>>(static_cast<const uint4 *>(k_new),
                                                    static_cast<const uint4 *>(v_new), static_cast<uint4 *>(kv_pool),
                                                    slots, hdr, n_kv_heads, cpv);
    return cudaGetLastError();
}

// Load the kernels now (CUDA lazy loading would otherwise load them at their first
// launch, which can block behind a spinning kernel such as apex_signal_wait's).
cudaError_t append_prepare() {
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, apex_append_kernel);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, apex_apply_deltas_kernel);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, apex_upload_kernel);
    return e;
}

}  // namespace apex
