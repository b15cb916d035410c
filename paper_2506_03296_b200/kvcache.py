"""PagedKVCache: torch-owned device memory + the C-ABI handle.

PyTorch supplies device memory (pools, block table, lengths, workspace) and the
current CUDA stream; the allocator, planner, append, decode attention and merge
all run inside libapex.so (include/apex.h).  A host-only cache (host_only=True)
runs the allocator/planner without any CUDA call (CPU tests, sharding logic).
"""
from __future__ import annotations

import contextlib
import ctypes
import math

import numpy as np

from . import apex as A

_TORCH_DT = {"f32": "float32", "f16": "float16", "bf16": "bfloat16"}


def torch_dtype(dtype: str):
    import torch
    return getattr(torch, _TORCH_DT[dtype])


def _stream_ptr(device) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream


class PagedKVCache:
    def __init__(self, *, num_layers: int, num_q_heads: int, num_kv_heads: int, num_blocks: int,
                 max_seqs: int, max_blocks_per_seq: int, max_batch: int, max_new_tokens: int,
                 dtype: str = "bf16", head_dim: int = 128, block_size: int = 16, device="cuda",
                 host_only: bool = False):
        self.num_layers, self.num_q_heads, self.num_kv_heads = num_layers, num_q_heads, num_kv_heads
        self.head_dim, self.block_size, self.dtype = head_dim, block_size, dtype
        self.num_blocks, self.max_seqs, self.max_blocks_per_seq = num_blocks, max_seqs, max_blocks_per_seq
        self.max_batch, self.max_new_tokens = max_batch, max_new_tokens
        self.host_only = host_only
        self.batch_seq_ids: list[int] = []
        self.n_rows = 0
        desc = A.apex_kv_desc(num_layers, num_q_heads, num_kv_heads, head_dim, block_size, num_blocks, max_seqs,
                              max_blocks_per_seq, max_batch, max_new_tokens, A.DTYPE_CODE[dtype])
        if host_only:
            self.device = None
            self.handle = A.apex_kv_create(desc)
            return
        import torch
        self.device = torch.device(device)
        if self.device.type == "cuda" and self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        tdt = torch_dtype(dtype)
        # one pool per physical layer: [num_blocks][Hkv][2 (K, V)][block_size][D]
        shape = (num_blocks, num_kv_heads, 2, block_size, head_dim)
        self.kv_pools = [torch.empty(shape, dtype=tdt, device=self.device) for _ in range(num_layers)]
        self.k_pools = [t[:, :, 0] for t in self.kv_pools]      # views [num_blocks][Hkv][16][D]
        self.v_pools = [t[:, :, 1] for t in self.kv_pools]
        self.block_table = torch.zeros((max_seqs, max_blocks_per_seq), dtype=torch.int32, device=self.device)
        self.seq_lens = torch.zeros((max_seqs,), dtype=torch.int32, device=self.device)
        desc.kv_pool = (ctypes.c_void_p * num_layers)(*[t.data_ptr() for t in self.kv_pools])
        desc.block_table, desc.seq_lens = self.block_table.data_ptr(), self.seq_lens.data_ptr()
        with torch.cuda.device(self.device):
            nbytes = A.apex_kv_workspace_bytes(desc)
            if nbytes == 0:
                # surface the validation message
                A.apex_kv_create(desc)
            self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            desc.workspace, desc.workspace_bytes = self.workspace.data_ptr(), nbytes
            self.handle = A.apex_kv_create(desc)

    # -- lifecycle
    def close(self):
        if getattr(self, "handle", None):
            A.apex_kv_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _stream(self) -> int:
        return 0 if self.host_only else _stream_ptr(self.device)

    def _on_device(self):
        """Make this cache's GPU current for an ABI call (the library uses the current
        device for attributes, memsets and the SM count)."""
        if self.host_only:
            return contextlib.nullcontext()
        import torch
        return torch.cuda.device(self.device)

    # -- step API (names follow the C ABI)
    def alloc(self, seq_ids, n_new):
        with self._on_device():
            A.apex_kv_alloc(self.handle, seq_ids, n_new, self._stream())
        self.batch_seq_ids = np.asarray(seq_ids, dtype=np.int64).tolist()
        self.n_rows = int(np.asarray(n_new, dtype=np.int64).sum())

    def release(self, seq_id: int):
        A.apex_kv_release(self.handle, seq_id)

    def append(self, layer: int, k_new, v_new):
        self._check_rows(k_new, self.n_rows, self.num_kv_heads)
        self._check_rows(v_new, self.n_rows, self.num_kv_heads)
        with self._on_device():
            A.apex_kv_append(self.handle, layer, k_new.data_ptr(), v_new.data_ptr(), self._stream())

    def decode(self, layer: int, q, out=None, scale: float | None = None):
        import torch
        B = len(self.batch_seq_ids)
        self._check_rows(q, B, self.num_q_heads)
        if out is None:
            out = torch.empty_like(q)
        else:
            self._check_rows(out, B, self.num_q_heads)
        if scale is None:
            scale = 1.0 / math.sqrt(self.head_dim)
        with self._on_device():
            A.apex_decode_attention(self.handle, layer, q.data_ptr(), out.data_ptr(), scale, self._stream())
        return out

    def decode_append(self, layer: int, q, k_new, v_new, out=None, scale: float | None = None):
        """append(layer, k_new, v_new) + decode(layer, q) in one launch (pure decode step:
        one new token per sequence).  Bit-identical to the two calls."""
        import torch
        B = len(self.batch_seq_ids)
        self._check_rows(q, B, self.num_q_heads)
        self._check_rows(k_new, B, self.num_kv_heads)
        self._check_rows(v_new, B, self.num_kv_heads)
        if out is None:
            out = torch.empty_like(q)
        else:
            self._check_rows(out, B, self.num_q_heads)
        if scale is None:
            scale = 1.0 / math.sqrt(self.head_dim)
        with self._on_device():
            A.apex_decode_attention_append(self.handle, layer, q.data_ptr(), k_new.data_ptr(), v_new.data_ptr(),
                                           out.data_ptr(), scale, self._stream())
        return out

    def decode_into(self, layer: int, q, outs, head_offset: int = 0, layout: str = "bhd", scale: float | None = None,
                    signals=None, signal_slot: int = 0, signal_value: int = 0):
        """Decode writing this handle's q heads into each tensor of `outs` at head `head_offset`.

        layout "bhd": outs are [B][H_total][D] (row-major); "hbd": [H_total][B][D]
        (head-major: a rank's head slice is contiguous, so an NCCL all-gather of
        [Hq/N][B][D] slices yields [Hq][B][D] with no permute).  All outs must have the
        same shape and dtype.  With peer-mapped symmetric buffers of the other ranks as
        `outs` the all-gather happens in the epilogue (f3); `signals` (one uint32 tensor
        or pointer per destination) then receive `signal_value` at `signal_slot` once
        every row is stored (in-kernel completion flag)."""
        B = len(self.batch_seq_ids)
        self._check_rows(q, B, self.num_q_heads)
        if not outs:
            raise ValueError("outs is empty")
        shape = tuple(outs[0].shape)
        want_dt = torch_dtype(self.dtype)
        for o in outs:
            if (tuple(o.shape) != shape or o.dim() != 3 or not o.is_contiguous() or o.dtype != want_dt
                    or o.device != self.device):
                raise ValueError("outs must be contiguous 3-D tensors of one shape and the cache dtype")
        if layout == "bhd":
            h_total = shape[1]
            if shape[0] != B or shape[2] != self.head_dim:
                raise ValueError(f"bhd outs must be [B={B}][H][{self.head_dim}], got {shape}")
            row_stride, head_stride = h_total * self.head_dim, self.head_dim
        elif layout == "hbd":
            h_total = shape[0]
            if shape[1] != B or shape[2] != self.head_dim:
                raise ValueError(f"hbd outs must be [H][B={B}][{self.head_dim}], got {shape}")
            row_stride, head_stride = self.head_dim, B * self.head_dim
        else:
            raise ValueError(f"unknown layout {layout!r}")
        if head_offset < 0 or head_offset + self.num_q_heads > h_total:
            raise ValueError(f"heads [{head_offset}, {head_offset + self.num_q_heads}) exceed H_total={h_total}")
        if scale is None:
            scale = 1.0 / math.sqrt(self.head_dim)
        sig = None
        if signals is not None:
            sig = [x if isinstance(x, int) else x.data_ptr() for x in signals]
        with self._on_device():
            A.apex_decode_attention_ex(self.handle, layer, q.data_ptr(), [o.data_ptr() for o in outs], row_stride,
                                       head_stride, head_offset, scale, self._stream(), sig, signal_slot,
                                       signal_value)

    def _check_rows(self, t, rows, heads):
        if t.device != self.device or t.dtype != torch_dtype(self.dtype) or not t.is_contiguous():
            raise ValueError(f"expected contiguous {self.dtype} tensor on {self.device}, got {t.dtype} on {t.device}")
        if tuple(t.shape) != (rows, heads, self.head_dim):
            raise ValueError(f"expected shape {(rows, heads, self.head_dim)}, got {tuple(t.shape)}")

    # -- knobs / introspection
    def set_split(self, chunk_tokens: int):
        A.apex_kv_set_split(self.handle, chunk_tokens)

    def set_grid(self, ctas: int):
        A.apex_kv_set_grid(self.handle, ctas)

    def plan_ranges(self):
        return A.apex_kv_plan_ranges(self.handle)

    def set_sched(self, dyn_permille: int):
        """-1: dynamic longest-first split items; 0..1000: stream-K static ranges with
        that permille of the tiles left to the dynamic queue (bandwidth regime)."""
        A.apex_kv_set_sched(self.handle, dyn_permille)

    def set_planner(self, latency_tiles_per_cta: int = 512, guided_div: int = 4, guided_pm=(900, 950, 980)):
        """Planner constants (tuning aid; include/apex.h apex_kv_set_planner)."""
        A.apex_kv_set_planner(self.handle, latency_tiles_per_cta, guided_div, *guided_pm)

    def num_free_blocks(self) -> int:
        return A.apex_kv_num_free_blocks(self.handle)

    def seq_info(self, seq_id: int):
        return A.apex_kv_seq_info(self.handle, seq_id)

    def last_slots(self):
        return A.apex_kv_last_slots(self.handle)

    def plan(self):
        return A.apex_kv_plan(self.handle)

    def decode_launches(self) -> int:
        """Kernel launches the next decode() issues (1, or 2 with the merge kernel)."""
        return A.apex_kv_decode_launches(self.handle)


def synth_rows(out, dtype: str, tensor: int, layer: int, row_b, row_pos, head_offset: int = 0, seed: int = 0,
               amp: float = 1.0):
    """Fill out [R][H][D] on the GPU with synth.gen_rows-identical values (device twin)."""
    import torch
    assert out.is_contiguous() and out.dim() == 3
    rb = row_b.to(device=out.device, dtype=torch.int32).contiguous()
    rp = row_pos.to(device=out.device, dtype=torch.int32).contiguous()
    A.apex_synth_rows(out.data_ptr(), dtype, tensor, layer, rb.data_ptr(), rp.data_ptr(), out.shape[0],
                      out.shape[1], head_offset, out.shape[2], seed, amp, _stream_ptr(out.device))
    return out
