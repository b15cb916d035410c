"""ORACLE (test infrastructure only) — Python front end of the float64 C oracle.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module.  The product package
``paper_2506_03296_b200`` never imports it.

``decode_attention`` is the plain definition of decode attention (SURVEY.md
§8(c); BASELINE.json north_star for the formula):
out[b,h,:] = softmax_t(scale * q[b,h,:].K[b,g(h),t,:]) . V[b,g(h),t,:] with
g(h) = h // (Hq/Hkv), computed in float64 over the LOGICAL contiguous cache by
``decode_attention_ref.c``.  See that file's header for the passages followed.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "decode_attention_ref.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_DT = {"f32": 0, "f16": 1, "bf16": 2, "f64": 3}
_NP = {"f32": np.float32, "f16": np.uint16, "bf16": np.uint16, "f64": np.float64}

_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle with plain gcc -O2 (no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fno-fast-math", "-fPIC", "-shared",
                               "-pthread", _SRC, "-o", _LIB, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.oracle_decode_attention.restype = ctypes.c_int
        _lib.oracle_decode_attention.argtypes = [
            ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p),
            ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_int64), ctypes.c_int,
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
            ctypes.POINTER(ctypes.c_int64), ctypes.c_int64, ctypes.c_void_p, ctypes.c_int]
        _lib.oracle_attention_weights.restype = ctypes.c_int
        _lib.oracle_attention_weights.argtypes = [
            ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
            ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_void_p]
        _lib.oracle_decode_f16.restype = ctypes.c_double
        _lib.oracle_decode_f16.argtypes = [ctypes.c_uint16]
        _lib.oracle_decode_bf16.restype = ctypes.c_double
        _lib.oracle_decode_bf16.argtypes = [ctypes.c_uint16]
    return _lib


def _check(a: np.ndarray, dtype: str) -> np.ndarray:
    a = np.ascontiguousarray(a)
    if a.dtype != _NP[dtype]:
        raise TypeError(f"oracle input for dtype {dtype} must be {_NP[dtype]}, got {a.dtype}")
    return a


def default_scale(head_dim: int) -> float:
    """1/sqrt(d) in double (reading c1)."""
    return 1.0 / math.sqrt(head_dim)


def decode_attention(q, ks, vs, dtype: str, scale: float | None = None, rows=None,
                     nthreads: int | None = None) -> np.ndarray:
    """Float64 decode attention.

    q:      [B][Hq][D] storage array of ``dtype`` (float32 / uint16 bits / float64)
    ks, vs: length-B lists of [n_b][Hkv][D] storage arrays (logical token order)
    rows:   optional int array of row ids b*Hq+h; default all rows
    returns [B][Hq][D] float64 (or [len(rows)][D] when ``rows`` is given)
    """
    q = _check(q, dtype)
    B, Hq, D = q.shape
    assert len(ks) == len(vs) == B
    ks = [_check(k, dtype) for k in ks]
    vs = [_check(v, dtype) for v in vs]
    Hkv = ks[0].shape[1] if B else 1
    for k, v in zip(ks, vs):
        assert k.shape == v.shape and k.shape[1:] == (Hkv, D), (k.shape, v.shape)
    n = np.array([k.shape[0] for k in ks], dtype=np.int64)
    kp = (ctypes.c_void_p * max(B, 1))(*[k.ctypes.data for k in ks])
    vp = (ctypes.c_void_p * max(B, 1))(*[v.ctypes.data for v in vs])
    if scale is None:
        scale = default_scale(D)
    if rows is None:
        out = np.empty((B, Hq, D), dtype=np.float64)
        rows_p, n_rows = None, B * Hq
    else:
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        out = np.empty((len(rows), D), dtype=np.float64)
        rows_p, n_rows = rows.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), len(rows)
    if nthreads is None:
        nthreads = len(os.sched_getaffinity(0))
    rc = lib().oracle_decode_attention(
        _DT[dtype], q.ctypes.data, kp, vp, n.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
        B, Hq, Hkv, D, float(scale), rows_p, n_rows, out.ctypes.data, int(nthreads))
    if rc != 0:
        raise ValueError(f"oracle_decode_attention rejected its arguments (rc={rc})")
    return out


def attention_weights(q_row, k, g: int, dtype: str, scale: float | None = None) -> np.ndarray:
    """Softmax weights w[t] of one query row q_row [D] against k [n][Hkv][D], kv head g."""
    q_row = _check(q_row, dtype)
    k = _check(k, dtype)
    n, Hkv, D = k.shape
    w = np.empty(n, dtype=np.float64)
    rc = lib().oracle_attention_weights(_DT[dtype], q_row.ctypes.data, k.ctypes.data, n, Hkv, g,
                                        D, float(default_scale(D) if scale is None else scale),
                                        w.ctypes.data)
    if rc != 0:
        raise ValueError("oracle_attention_weights rejected its arguments")
    return w


def decode_element(bits: int, dtype: str) -> float:
    """The oracle's own fp16/bf16 field decoder (pinned against numpy in tests)."""
    return lib().oracle_decode_f16(bits) if dtype == "f16" else lib().oracle_decode_bf16(bits)
