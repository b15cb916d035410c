"""Partitioning of the decode-attention work across the GPUs of one box.

Every (request, kv head) attention is independent, so:
  * request sharding: requests are split across ranks (greedy LPT on context
    length so ragged batches balance their KV bytes); no collective;
  * head sharding: rank r owns kv heads [r*Hkv/N, (r+1)*Hkv/N) and their
    q-groups for every request; the only collective is an all-gather of the
    attention outputs (NCCL over NVLink in production, gloo in CPU tests).
Host logic only; the attention itself runs in libapex.so on each rank.
"""
from __future__ import annotations

import heapq


def lpt_partition(lengths, n_ranks: int):
    """Greedy longest-processing-time assignment of requests to ranks.

    Returns a list (per rank) of request indices, each in ascending order.
    Deterministic: ties broken by request index and rank index."""
    if n_ranks < 1:
        raise ValueError("n_ranks must be >= 1")
    order = sorted(range(len(lengths)), key=lambda i: (-int(lengths[i]), i))
    heap = [(0, r) for r in range(n_ranks)]
    parts = [[] for _ in range(n_ranks)]
    for i in order:
        load, r = heapq.heappop(heap)
        parts[r].append(i)
        heapq.heappush(heap, (load + int(lengths[i]), r))
    return [sorted(p) for p in parts]


def head_range(num_kv_heads: int, num_q_heads: int, rank: int, world: int):
    """(kv_lo, kv_hi, q_lo, q_hi) owned by `rank` under head sharding."""
    if num_kv_heads % world:
        raise ValueError(f"{num_kv_heads} kv heads cannot be split over {world} ranks")
    g = num_q_heads // num_kv_heads
    per = num_kv_heads // world
    return rank * per, (rank + 1) * per, rank * per * g, (rank + 1) * per * g


def symmetric_output(shape, dtype, device, group=None):
    """A full-width output buffer in torch symmetric memory + its rendezvous handle.

    handle.buffer_ptrs holds every rank's (peer-mapped) address of its buffer, to
    be passed as the destinations of apex_decode_attention_ex: each rank then
    stores its head slice into all ranks' buffers from the kernel epilogue (the
    all-gather fused into the decode); handle.barrier()
    orders those remote stores before the gathered rows are read.
    NOTE: exercised on one GPU only with local destinations
    (tests/test_fused_gather_gpu.py); the peer-pointer path needs >= 2 GPUs."""
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm_mem
    t = symm_mem.empty(*shape, dtype=dtype, device=device)
    handle = symm_mem.rendezvous(t, group if group is not None else dist.group.WORLD)
    return t, handle


def gather_heads(out_local, group=None):
    """All-gather head-sharded outputs [B][Hq/N][D] -> [B][Hq][D] view.

    all_gather_into_tensor lays the rank slices out as [N][B][Hq/N][D]; the
    returned tensor is the zero-copy permuted view [B][N][Hq/N][D] -> [B][Hq][D]
    is materialised only if the caller needs contiguity."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    B, hl, D = out_local.shape
    full = torch.empty((world * B, hl, D), dtype=out_local.dtype, device=out_local.device)
    dist.all_gather_into_tensor(full, out_local.contiguous(), group=group)
    return full.view(world, B, hl, D).permute(1, 0, 2, 3).reshape(B, world * hl, D)
