"""Workload recipes for BASELINE.json configs C1..C5 (shapes only; no method arithmetic).

Each recipe gives the attention shape, dtype, logical layer count and the
per-request context length ``ctx[b]`` = tokens the request attends over at the
FIRST decode step (prefill writes ctx[b]-1 tokens, the step appends one more).
See DESIGN.md "Input recipe" and SURVEY.md §8(d).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .gen import splitmix64


@dataclass(frozen=True)
class Workload:
    name: str
    desc: str
    batch: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    dtype: str
    layers: int
    ctx_kind: str                 # "uniform" | "hash" | "skew"
    ctx: int = 0                  # uniform context
    ctx_lo: int = 1024            # hash draw: lo + splitmix64(b) % span
    ctx_span: int = 31745
    steps: int = 1                # decode steps the recipe describes
    block_size: int = 16
    extra: dict = field(default_factory=dict)

    @property
    def group(self) -> int:
        return self.num_q_heads // self.num_kv_heads

    def contexts(self, batch: int | None = None, b0: int = 0) -> np.ndarray:
        """ctx[b] for requests b0 .. b0+batch-1 (global request ids)."""
        n = self.batch if batch is None else batch
        b = np.arange(b0, b0 + n, dtype=np.uint64)
        if self.ctx_kind == "uniform":
            return np.full(n, self.ctx, dtype=np.int64)
        if self.ctx_kind == "skew":                     # request 0 long, the rest short
            return np.where(b == 0, self.ctx, self.ctx_lo).astype(np.int64)
        return (self.ctx_lo + (splitmix64(b) % np.uint64(self.ctx_span))).astype(np.int64)


WORKLOADS = {
    "c1": Workload("c1", "1 layer, batch 1, 32 heads, head_dim 128, context 512, fp32 KV",
                   1, 32, 32, 128, "f32", 1, "uniform", ctx=512),
    "c2": Workload("c2", "LLaMA-2-7B MHA decode, batch 64, uniform context 4K, 32 layers, fp16 paged KV (block 16)",
                   64, 32, 32, 128, "f16", 32, "uniform", ctx=4096),
    "c3": Workload("c3", "LLaMA-3.1-8B GQA (32 q / 8 kv heads) decode, batch 128, context 8K, bf16 paged KV",
                   128, 32, 8, 128, "bf16", 32, "uniform", ctx=8192),
    "c4": Workload("c4", "long-output CoT mix: batch 256, ragged contexts 1K-32K, LLaMA-3.1-8B GQA, bf16, continuous kv_append per step",
                   256, 32, 8, 128, "bf16", 32, "hash", steps=64),
    # load-balance stress variant of C4: 1 x 32K + 255 x 1K; not a BASELINE config
    "c4s": Workload("c4s", "C4 skew variant: batch 256, one 32K context + 255 x 1K, LLaMA-3.1-8B GQA, bf16",
                    256, 32, 8, 128, "bf16", 32, "skew", ctx=32768, ctx_lo=1024),
    "c5": Workload("c5", "LLaMA-3.1-8B GQA, batch 1024, context 16K, all 32 layers, sharded across 1/2/4/8 B200",
                   1024, 32, 8, 128, "bf16", 32, "uniform", ctx=16384),
}


def kv_bytes_per_token_layer(w: Workload) -> int:
    """K+V bytes one token occupies in one layer."""
    es = 4 if w.dtype == "f32" else 2
    return 2 * w.num_kv_heads * w.head_dim * es
