"""Thin ctypes binding of the C ABI (include/apex.h, include/apex_synth.h).

Argument marshalling only: every step of the hot path runs in libapex.so's
kernels.  Function names match the C entry points; non-OK statuses raise
ApexError carrying apex_last_error().  There is no fallback: if libapex.so is
missing this module raises (build it with ``python -m
paper_2506_03296_b200.build`` or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_int32, c_int64, c_size_t, c_uint32, c_uint64, c_void_p

LIB_PATH = os.environ.get("APEX_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libapex.so")

APEX_OK, APEX_EINVAL, APEX_ENOBLOCKS, APEX_ESEQ, APEX_ECUDA, APEX_EUNSUPPORTED = range(6)
STATUS_NAMES = {0: "APEX_OK", 1: "APEX_EINVAL", 2: "APEX_ENOBLOCKS", 3: "APEX_ESEQ", 4: "APEX_ECUDA",
                5: "APEX_EUNSUPPORTED"}
APEX_F32, APEX_F16, APEX_BF16 = 0, 1, 2
DTYPE_CODE = {"f32": APEX_F32, "f16": APEX_F16, "bf16": APEX_BF16}

# every symbol the public headers declare (checked by tests/test_host_core.py)
EXPORTS = ["apex_kv_workspace_bytes", "apex_kv_create", "apex_kv_destroy", "apex_kv_alloc", "apex_kv_release",
           "apex_kv_append", "apex_decode_attention", "apex_kv_set_split", "apex_kv_set_grid", "apex_kv_set_sched",
           "apex_kv_num_free_blocks", "apex_kv_seq_info", "apex_kv_last_slots", "apex_kv_plan", "apex_kv_plan_ranges",
           "apex_cost_create", "apex_predict_time", "apex_cost_destroy", "apex_last_error", "apex_version",
           "apex_synth_rows", "apex_pipelining_threshold", "apex_decide", "apex_kv_decode_launches", "apex_decode_attention_ex",
           "apex_decode_attention_append", "apex_signal_wait", "apex_signal_post", "apex_cost_observe",
           "apex_cost_size", "apex_cost_table", "apex_kv_set_planner"]
STRATEGIES = {0: "gpu_only", 1: "asym_pipeline", 2: "async_overlap"}


class ApexError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.code = STATUS_NAMES.get(status, str(status)).replace("APEX_", "")


class apex_kv_desc(ctypes.Structure):
    _fields_ = [("num_layers", c_int32), ("num_q_heads", c_int32), ("num_kv_heads", c_int32),
                ("head_dim", c_int32), ("block_size", c_int32), ("num_blocks", c_int32), ("max_seqs", c_int32),
                ("max_blocks_per_seq", c_int32), ("max_batch", c_int32), ("max_new_tokens", c_int32),
                ("dtype", c_int), ("kv_pool", POINTER(c_void_p)),
                ("block_table", c_void_p), ("seq_lens", c_void_p), ("workspace", c_void_p),
                ("workspace_bytes", c_size_t)]


class apex_sched_input(ctypes.Structure):
    _fields_ = [("n_prefill", c_int32), ("n_gpu_decode", c_int32), ("n_cpu_decode", c_int32), ("n_g", c_double),
                ("n_c", c_double), ("t_glinear", c_double), ("t_gatt", c_double), ("t_glinear_pref", c_double),
                ("t_gatt_pref", c_double), ("min_cpu_ratio", c_double)]


class apex_decision(ctypes.Structure):
    _fields_ = [("strategy", c_int), ("gate_closed", c_int32), ("lhs", c_double), ("rhs", c_double),
                ("eq6_threshold", c_double)]


_lib = None


def lib():
    """Load libapex.so (raises if it was not built -- no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2506_03296_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        P32 = POINTER(c_int32)
        sig = {
            "apex_kv_workspace_bytes": (c_size_t, [POINTER(apex_kv_desc)]),
            "apex_kv_create": (c_int, [POINTER(apex_kv_desc), POINTER(c_void_p)]),
            "apex_kv_destroy": (None, [c_void_p]),
            "apex_kv_alloc": (c_int, [c_void_p, P32, P32, c_int32, c_void_p]),
            "apex_kv_release": (c_int, [c_void_p, c_int32]),
            "apex_kv_append": (c_int, [c_void_p, c_int32, c_void_p, c_void_p, c_void_p]),
            "apex_decode_attention": (c_int, [c_void_p, c_int32, c_void_p, c_void_p, c_float, c_void_p]),
            "apex_kv_set_split": (c_int, [c_void_p, c_int32]),
            "apex_kv_set_grid": (c_int, [c_void_p, c_int32]),
            "apex_kv_set_sched": (c_int, [c_void_p, c_int32]),
            "apex_kv_num_free_blocks": (c_int32, [c_void_p]),
            "apex_kv_seq_info": (c_int, [c_void_p, c_int32, P32, P32, c_int32, P32]),
            "apex_kv_last_slots": (c_int, [c_void_p, P32, c_int32, P32]),
            "apex_kv_plan": (c_int, [c_void_p, P32, c_int32, P32, P32]),
            "apex_kv_plan_ranges": (c_int, [c_void_p, P32, c_int32, P32]),
            "apex_cost_create": (c_int, [P32, c_int32, POINTER(c_int64), c_int32, POINTER(c_double),
                                         POINTER(c_void_p)]),
            "apex_predict_time": (c_int, [c_void_p, c_int32, c_int64, POINTER(c_double)]),
            "apex_cost_destroy": (None, [c_void_p]),
            "apex_last_error": (c_char_p, []),
            "apex_version": (c_char_p, []),
            "apex_synth_rows": (c_int, [c_void_p, c_int, c_int32, c_int32, c_void_p, c_void_p, c_int64, c_int32,
                                        c_int32, c_int32, c_uint64, c_float, c_void_p]),
            "apex_pipelining_threshold": (c_int, [c_double, c_double, POINTER(c_double)]),
            "apex_decide": (c_int, [POINTER(apex_sched_input), POINTER(apex_decision)]),
            "apex_kv_decode_launches": (c_int32, [c_void_p]),
            "apex_decode_attention_ex": (c_int, [c_void_p, c_int32, c_void_p, POINTER(c_void_p), c_int32, c_int64,
                                                 c_int64, c_int32, POINTER(c_void_p), c_int32, c_uint32, c_float,
                                                 c_void_p]),
            "apex_kv_set_planner": (c_int, [c_void_p, c_int32, c_int32, c_int32, c_int32, c_int32]),
            "apex_cost_observe": (c_int, [c_void_p, c_int32, c_int64, c_double, c_double]),
            "apex_cost_size": (c_int, [c_void_p, POINTER(c_int32), POINTER(c_int32)]),
            "apex_cost_table": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
            "apex_signal_wait": (c_int, [c_void_p, c_int32, c_uint32, c_uint64, c_void_p, c_void_p]),
            "apex_signal_post": (c_int, [POINTER(c_void_p), c_int32, c_int32, c_uint32, c_void_p]),
            "apex_decode_attention_append": (c_int, [c_void_p, c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
                                                     c_float, c_void_p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def _check(status: int):
    if status != APEX_OK:
        raise ApexError(status, lib().apex_last_error().decode())


def _i32(seq):
    """int32 C array of `seq` (list, tuple or array); the returned pointer keeps the
    numpy buffer alive for the call (numpy: ~10x faster than a ctypes array built
    from Python ints for batch-sized lists)."""
    arr = np.ascontiguousarray(seq, dtype=np.int32)
    if arr.size == 0:
        arr = np.zeros(1, dtype=np.int32)
    return arr.ctypes.data_as(ctypes.POINTER(c_int32))


# ------------------------------------------------------------------ C-ABI mirrors

def apex_version() -> str:
    return lib().apex_version().decode()


def apex_kv_workspace_bytes(desc: apex_kv_desc) -> int:
    return int(lib().apex_kv_workspace_bytes(ctypes.byref(desc)))


def apex_kv_create(desc: apex_kv_desc) -> int:
    h = c_void_p()
    _check(lib().apex_kv_create(ctypes.byref(desc), ctypes.byref(h)))
    return h.value


def apex_kv_destroy(kv: int) -> None:
    lib().apex_kv_destroy(kv)


def apex_kv_alloc(kv: int, seq_ids, n_new, stream: int = 0) -> None:
    assert len(seq_ids) == len(n_new)
    _check(lib().apex_kv_alloc(kv, _i32(seq_ids), _i32(n_new), len(seq_ids), stream))


def apex_kv_release(kv: int, seq_id: int) -> None:
    _check(lib().apex_kv_release(kv, int(seq_id)))


def apex_kv_append(kv: int, layer: int, k_new_ptr: int, v_new_ptr: int, stream: int = 0) -> None:
    _check(lib().apex_kv_append(kv, int(layer), k_new_ptr, v_new_ptr, stream))


def apex_decode_attention(kv: int, layer: int, q_ptr: int, out_ptr: int, scale: float, stream: int = 0) -> None:
    _check(lib().apex_decode_attention(kv, int(layer), q_ptr, out_ptr, float(scale), stream))


def apex_decode_attention_append(kv: int, layer: int, q_ptr: int, k_ptr: int, v_ptr: int, out_ptr: int,
                                 scale: float, stream: int = 0) -> None:
    _check(lib().apex_decode_attention_append(kv, int(layer), q_ptr, k_ptr, v_ptr, out_ptr, float(scale), stream))


def apex_kv_set_split(kv: int, chunk_tokens: int) -> None:
    _check(lib().apex_kv_set_split(kv, int(chunk_tokens)))


def apex_kv_set_grid(kv: int, ctas: int) -> None:
    _check(lib().apex_kv_set_grid(kv, int(ctas)))


def apex_kv_set_sched(kv: int, dyn_permille: int) -> None:
    _check(lib().apex_kv_set_sched(kv, int(dyn_permille)))


def apex_kv_set_planner(kv: int, latency_tiles_per_cta: int = 512, guided_div: int = 8, guided_pm1: int = 900,
                        guided_pm2: int = 950, guided_pm3: int = 980) -> None:
    _check(lib().apex_kv_set_planner(kv, int(latency_tiles_per_cta), int(guided_div), int(guided_pm1),
                                     int(guided_pm2), int(guided_pm3)))


def apex_kv_num_free_blocks(kv: int) -> int:
    return int(lib().apex_kv_num_free_blocks(kv))


def apex_kv_seq_info(kv: int, seq_id: int):
    """(len, [block ids in table order])"""
    ln, nb = c_int32(), c_int32()
    _check(lib().apex_kv_seq_info(kv, int(seq_id), ctypes.byref(ln), None, 0, ctypes.byref(nb)))
    buf = (c_int32 * max(nb.value, 1))()
    _check(lib().apex_kv_seq_info(kv, int(seq_id), ctypes.byref(ln), buf, nb.value, ctypes.byref(nb)))
    return ln.value, list(buf[:nb.value])


def apex_kv_last_slots(kv: int):
    n = c_int32()
    _check(lib().apex_kv_last_slots(kv, None, 0, ctypes.byref(n)))
    buf = (c_int32 * max(n.value, 1))()
    _check(lib().apex_kv_last_slots(kv, buf, n.value, ctypes.byref(n)))
    return list(buf[:n.value])


def apex_kv_plan_ranges(kv: int):
    """Per-CTA static item ranges of the last plan: list of grid + 1 offsets."""
    n = c_int32(0)
    _check(lib().apex_kv_plan_ranges(kv, None, 0, ctypes.byref(n)))
    buf = (c_int32 * n.value)()
    _check(lib().apex_kv_plan_ranges(kv, buf, n.value, ctypes.byref(n)))
    return list(buf)


def apex_kv_plan(kv: int):
    """(items as list of (b, g, blk0, nblk, part, seq), n_merges)"""
    ni, nm = c_int32(), c_int32()
    _check(lib().apex_kv_plan(kv, None, 0, ctypes.byref(ni), ctypes.byref(nm)))
    buf = (c_int32 * max(6 * ni.value, 1))()
    _check(lib().apex_kv_plan(kv, buf, ni.value, ctypes.byref(ni), ctypes.byref(nm)))
    flat = list(buf[:6 * ni.value])
    return [tuple(flat[6 * i:6 * i + 6]) for i in range(ni.value)], nm.value


def apex_cost_create(batch_grid, kv_grid, us) -> int:
    nb, nk = len(batch_grid), len(kv_grid)
    flat = [float(x) for row in us for x in row]
    assert len(flat) == nb * nk
    h = c_void_p()
    _check(lib().apex_cost_create(_i32(batch_grid), nb, (c_int64 * max(nk, 1))(*[int(x) for x in kv_grid]), nk,
                                  (c_double * max(len(flat), 1))(*flat), ctypes.byref(h)))
    return h.value


def apex_predict_time(cost: int, batch: int, kv_tokens: int) -> float:
    out = c_double()
    _check(lib().apex_predict_time(cost, int(batch), int(kv_tokens), ctypes.byref(out)))
    return out.value


def apex_cost_observe(cost: int, batch: int, kv_tokens: int, measured_us: float, alpha: float = 1.0) -> None:
    _check(lib().apex_cost_observe(cost, int(batch), int(kv_tokens), float(measured_us), float(alpha)))


def apex_cost_table(cost: int):
    """(batch_grid, kv_grid, us[nb][nk]) of the current table."""
    nb, nk = c_int32(), c_int32()
    _check(lib().apex_cost_size(cost, ctypes.byref(nb), ctypes.byref(nk)))
    bg, kg, us = (c_int32 * nb.value)(), (c_int64 * nk.value)(), (c_double * (nb.value * nk.value))()
    _check(lib().apex_cost_table(cost, bg, kg, us))
    return list(bg), list(kg), [list(us[i * nk.value:(i + 1) * nk.value]) for i in range(nb.value)]


def apex_cost_destroy(cost: int) -> None:
    lib().apex_cost_destroy(cost)


def apex_synth_rows(out_ptr: int, dtype: str, tensor: int, layer: int, row_b_ptr: int, row_pos_ptr: int,
                    n_rows: int, n_heads: int, head_offset: int, head_dim: int, seed: int, amp: float,
                    stream: int = 0) -> None:
    _check(lib().apex_synth_rows(out_ptr, DTYPE_CODE[dtype], tensor, layer, row_b_ptr, row_pos_ptr, n_rows,
                                 n_heads, head_offset, head_dim, seed, amp, stream))


def apex_pipelining_threshold(t_glinear: float, t_gatt: float) -> float:
    out = c_double()
    st = lib().apex_pipelining_threshold(float(t_glinear), float(t_gatt), ctypes.byref(out))
    _check(st)
    return out.value


def apex_decide(n_prefill: int, n_gpu_decode: int, n_cpu_decode: int, n_g: float, n_c: float, t_glinear: float,
                t_gatt: float, t_glinear_pref: float = 0.0, t_gatt_pref: float = 0.0, min_cpu_ratio: float = 8.0):
    """Algorithm 1 decision -> dict(strategy, gate_closed, lhs, rhs, eq6_threshold)."""
    inp = apex_sched_input(n_prefill, n_gpu_decode, n_cpu_decode, n_g, n_c, t_glinear, t_gatt, t_glinear_pref,
                           t_gatt_pref, min_cpu_ratio)
    out = apex_decision()
    st = lib().apex_decide(ctypes.byref(inp), ctypes.byref(out))
    _check(st)
    return {"strategy": STRATEGIES[out.strategy], "gate_closed": bool(out.gate_closed), "lhs": out.lhs,
            "rhs": out.rhs, "eq6_threshold": out.eq6_threshold}


def apex_kv_decode_launches(kv: int) -> int:
    return int(lib().apex_kv_decode_launches(kv))


def apex_decode_attention_ex(kv: int, layer: int, q_ptr: int, out_ptrs, out_row_stride: int, out_head_stride: int,
                             out_head_offset: int, scale: float, stream: int = 0, signal_ptrs=None,
                             signal_slot: int = 0, signal_value: int = 0) -> None:
    outs = (c_void_p * max(len(out_ptrs), 1))(*[int(x) for x in out_ptrs])
    sig = None
    if signal_ptrs is not None:
        if len(signal_ptrs) != len(out_ptrs):
            raise ValueError("one signal array per destination")
        sig = (c_void_p * len(signal_ptrs))(*[int(x) for x in signal_ptrs])
    _check(lib().apex_decode_attention_ex(kv, int(layer), q_ptr, outs, len(out_ptrs), int(out_row_stride),
                                          int(out_head_stride), int(out_head_offset), sig, int(signal_slot),
                                          int(signal_value) & 0xffffffff, float(scale), stream))


def apex_signal_wait(signals_ptr: int, n: int, value: int, timeout_ns: int, status_ptr: int = 0,
                     stream: int = 0) -> None:
    _check(lib().apex_signal_wait(signals_ptr, int(n), int(value) & 0xffffffff, int(timeout_ns), status_ptr or None,
                                  stream))


def apex_signal_post(dst_ptrs, slot: int, value: int, stream: int = 0) -> None:
    dst = (c_void_p * max(len(dst_ptrs), 1))(*[int(x) for x in dst_ptrs])
    _check(lib().apex_signal_post(dst, len(dst_ptrs), int(slot), int(value) & 0xffffffff, stream))
