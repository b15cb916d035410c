"""Seeded synthetic inputs shared by the oracle side and the CUDA side (no method arithmetic)."""
from .gen import (TENSOR_Q, TENSOR_K, TENSOR_V, DTYPES, DTYPE_CODE, ELEM_BYTES, LIMITS,
                  splitmix64, splitmix64_int, make_key, gen_f32, gen_rows, gen_seq, encode,
                  f32_to_bf16_bits, f32_to_f16_bits)
from .workloads import WORKLOADS, Workload, kv_bytes_per_token_layer
