/*
 * apex_synth.h — device twin of the seeded input generator (synth/gen.py).
 *
 * Test/bench utility, not part of the method: it fills device buffers with the
 * same values synth.gen_rows() produces on the host, so multi-GiB KV caches
 * can be created on the GPU and any row regenerated on the host for the
 * oracle without reading device memory (SURVEY.md §8(d) "Synthetic inputs").
 *
 *   rowkey = tensor<<55 | layer<<49 | b<<33 | head<<26 | t<<8
 *   hrow   = splitmix64(rowkey ^ splitmix64(seed))
 *   u      = lowbias32(lo32(hrow) + d * 0x9E3779B9) ^ hi32(hrow)
 *   x      = ((u>>8) - 2^23) * 2^-22 * amp
 *   stored as fp32, or rounded to nearest even to fp16 / bf16.
 */
#ifndef APEX_SYNTH_H
#define APEX_SYNTH_H

#include "apex.h"

#ifdef __cplusplus
extern "C" {
#endif

/* out: device [n_rows][n_heads][head_dim] of dtype.  row_b, row_pos: device
   int32 [n_rows] (request id and token position of each row).  Head h of the
   output is global head head_offset + h.  amp must be a power of two. */
apex_status apex_synth_rows(void *out, apex_dtype dtype, int32_t tensor, int32_t layer,
                            const int32_t *row_b, const int32_t *row_pos, int64_t n_rows,
                            int32_t n_heads, int32_t head_offset, int32_t head_dim,
                            uint64_t seed, float amp, apex_stream stream);

#ifdef __cplusplus
}
#endif
#endif
