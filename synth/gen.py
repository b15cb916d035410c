"""Seeded, counter-based synthetic input generator (host twin).

This module is shared by the oracle side (tests, bench cpu_baseline) and the
product side's tests/bench.  It holds NONE of the method's arithmetic: it only
produces input values (q, K, V rows) and workload shapes.  The CUDA twin lives
in ``paper_2506_03296_b200/csrc/synth.cu`` (``apex_synth_rows``); both
implement the same generator independently and ``tests/test_generator.py``
checks them bit-for-bit.

Generator (SURVEY.md §8(d) "Synthetic inputs"):

    rowkey = tensor<<55 | layer<<49 | b<<33 | head<<26 | t<<8      (the d field is 0)
    hrow   = splitmix64(rowkey XOR splitmix64(seed))             # one per (row, head)
    u      = lowbias32(lo32(hrow) + d * 0x9E3779B9) XOR hi32(hrow)  # uint32 arithmetic
    x      = ((u >> 8) - 2**23) * 2**-22          # exact in fp32, uniform [-2, 2)
    x16    = round-to-nearest-even(x * amp)       # fp16 / bf16 bit patterns

lowbias32 is Wellons' 32-bit integer finaliser (x ^= x>>16; x *= 0x7feb352d;
x ^= x>>15; x *= 0x846ca68b; x ^= x>>16).  One 64-bit mix per 128-dim row keeps
the device fill of 100+ GiB caches cheap.

``amp`` is a power of two (q x1, x8, x64 variants), so ``x * amp`` is exact in
fp32.  Values are keyed by logical (tensor, layer, request b, head, position t,
dim d) so any single row can be regenerated without reading device memory.
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
TENSOR_Q, TENSOR_K, TENSOR_V = 0, 1, 2

# field widths of the key (bits)
_D_BITS, _T_BITS, _H_BITS, _B_BITS, _L_BITS = 8, 18, 7, 16, 6
_T_SHIFT = _D_BITS
_H_SHIFT = _T_SHIFT + _T_BITS
_B_SHIFT = _H_SHIFT + _H_BITS
_L_SHIFT = _B_SHIFT + _B_BITS
_X_SHIFT = _L_SHIFT + _L_BITS          # tensor id

LIMITS = dict(d=1 << _D_BITS, t=1 << _T_BITS, head=1 << _H_BITS,
              b=1 << _B_BITS, layer=1 << _L_BITS, tensor=4)


def splitmix64_int(x: int) -> int:
    """Scalar splitmix64 finaliser (Steele/Lea/Flood; Vigna's reference constants)."""
    z = (x + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 over uint64 arrays (numpy uint64 arithmetic wraps mod 2**64)."""
    z = np.asarray(x, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def make_key(tensor, layer, b, head, t, d) -> np.ndarray:
    u = lambda v: np.asarray(v, dtype=np.uint64)
    return (u(tensor) << np.uint64(_X_SHIFT)) | (u(layer) << np.uint64(_L_SHIFT)) | \
           (u(b) << np.uint64(_B_SHIFT)) | (u(head) << np.uint64(_H_SHIFT)) | \
           (u(t) << np.uint64(_T_SHIFT)) | u(d)


def lowbias32(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint32)
    x = x ^ (x >> np.uint32(16))
    x = x * np.uint32(0x7FEB352D)
    x = x ^ (x >> np.uint32(15))
    x = x * np.uint32(0x846CA68B)
    return x ^ (x >> np.uint32(16))


def gen_f32(tensor, layer, b, head, t, d, seed: int = 0, amp: float = 1.0) -> np.ndarray:
    """fp32 values for broadcastable index arrays (exact: 24-bit lattice times a power of two)."""
    hrow = splitmix64(make_key(tensor, layer, b, head, t, 0) ^ np.uint64(splitmix64_int(seed)))
    lo = (hrow & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    hi = (hrow >> np.uint64(32)).astype(np.uint32)
    with np.errstate(over="ignore"):
        u = lowbias32(lo + np.asarray(d, dtype=np.uint32) * np.uint32(0x9E3779B9)) ^ hi
    v = (u >> np.uint32(8)).astype(np.int64) - (1 << 23)
    return (v.astype(np.float32) * np.float32(2.0 ** -22)) * np.float32(amp)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit pattern (inputs are finite)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = (u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return r.astype(np.uint16)


def f32_to_f16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> IEEE binary16 bit pattern (numpy's cast is RNE)."""
    return np.ascontiguousarray(x, dtype=np.float32).astype(np.float16).view(np.uint16)


DTYPES = ("f32", "f16", "bf16")
DTYPE_CODE = {"f32": 0, "f16": 1, "bf16": 2}      # matches apex_dtype in include/apex.h
ELEM_BYTES = {"f32": 4, "f16": 2, "bf16": 2}


def encode(x32: np.ndarray, dtype: str) -> np.ndarray:
    """fp32 values -> storage array (float32, or uint16 bit patterns for 16-bit types)."""
    if dtype == "f32":
        return np.ascontiguousarray(x32, dtype=np.float32)
    if dtype == "bf16":
        return f32_to_bf16_bits(x32)
    if dtype == "f16":
        return f32_to_f16_bits(x32)
    raise ValueError(dtype)


def gen_rows(tensor: int, layer: int, b, pos, n_heads: int, head_dim: int, dtype: str,
             seed: int = 0, amp: float = 1.0, head_offset: int = 0) -> np.ndarray:
    """Rows [R][n_heads][head_dim] for row r = (request b[r], position pos[r]).

    Heads are numbered globally from ``head_offset`` (head-sharded ranks generate
    their slice of the global tensor).
    """
    b = np.asarray(b, dtype=np.int64).reshape(-1, 1, 1)
    pos = np.asarray(pos, dtype=np.int64).reshape(-1, 1, 1)
    h = np.arange(head_offset, head_offset + n_heads, dtype=np.int64).reshape(1, -1, 1)
    d = np.arange(head_dim, dtype=np.int64).reshape(1, 1, -1)
    return encode(gen_f32(tensor, layer, b, h, pos, d, seed, amp), dtype)


def gen_seq(tensor: int, layer: int, b: int, n_tokens: int, n_heads: int, head_dim: int,
            dtype: str, seed: int = 0, amp: float = 1.0, head_offset: int = 0,
            t0: int = 0) -> np.ndarray:
    """Contiguous logical K or V of one request: [n_tokens][n_heads][head_dim]."""
    pos = np.arange(t0, t0 + n_tokens, dtype=np.int64)
    return gen_rows(tensor, layer, np.full(n_tokens, b), pos, n_heads, head_dim, dtype,
                    seed, amp, head_offset)
