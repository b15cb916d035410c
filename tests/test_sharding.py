"""Multi-GPU host logic on CPU: request (LPT) and kv-head partitioning, and the
head-sharded all-gather, with a world-size-2 gloo process group.

Per-rank attention here is the float64 oracle on the rank's slice (no GPU on
this box); the sharded-then-gathered result must equal the unsharded one
bit-for-bit, because every (request, q-head) row is computed independently.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import synth
from paper_2506_03296_b200.sharding import head_range, lpt_partition


def test_lpt_partition_covers_and_balances():
    rnd = np.random.default_rng(0)
    for n in (1, 2, 3, 8):
        lens = [int(x) for x in synth.WORKLOADS["c4"].contexts()]
        parts = lpt_partition(lens, n)
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(len(lens)))
        loads = [sum(lens[i] for i in p) for p in parts]
        assert max(loads) - min(loads) <= max(lens)
        assert parts == lpt_partition(lens, n)           # deterministic
    assert lpt_partition([5, 5, 5, 5], 2) == [[0, 2], [1, 3]]
    with pytest.raises(ValueError):
        lpt_partition([1], 0)


def test_head_range_partitions_heads():
    for world in (1, 2, 4, 8):
        kv, q = set(), set()
        for r in range(world):
            a, b, c, d = head_range(8, 32, r, world)
            assert d - c == 4 * (b - a)
            kv |= set(range(a, b))
            q |= set(range(c, d))
        assert kv == set(range(8)) and q == set(range(32))
    with pytest.raises(ValueError):
        head_range(8, 32, 0, 3)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, result_path):
    import torch
    import torch.distributed as dist

    from oracle import attention as oa
    from paper_2506_03296_b200.sharding import gather_heads, head_range, lpt_partition
    from paper_2506_03296_b200.kvcache import PagedKVCache

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    B, Hq, Hkv, D = 6, 8, 4, 128
    ctx = [3, 40, 17, 100, 1, 64]
    if mode == "head":
        kv_lo, kv_hi, q_lo, q_hi = head_range(Hkv, Hq, rank, world)
        q = synth.gen_rows(0, 0, range(B), [c - 1 for c in ctx], q_hi - q_lo, D, "bf16", head_offset=q_lo)
        ks = [synth.gen_seq(1, 0, b, c, kv_hi - kv_lo, D, "bf16", head_offset=kv_lo) for b, c in enumerate(ctx)]
        vs = [synth.gen_seq(2, 0, b, c, kv_hi - kv_lo, D, "bf16", head_offset=kv_lo) for b, c in enumerate(ctx)]
        local = torch.from_numpy(oa.decode_attention(q, ks, vs, "bf16", nthreads=1))
        # head-major [Hq/N][B][D] slices gather into [Hq][B][D] with no permute
        full = gather_heads(local.permute(1, 0, 2).contiguous())
        assert full.shape == (Hq, B, D)
        full = full.permute(1, 0, 2)
        # the rank's planner over its head slice covers exactly its kv heads
        cache = PagedKVCache(num_layers=1, num_q_heads=q_hi - q_lo, num_kv_heads=kv_hi - kv_lo, num_blocks=64,
                             max_seqs=B, max_blocks_per_seq=16, max_batch=B, max_new_tokens=1024, host_only=True)
        cache.alloc(list(range(B)), ctx)
        items, _ = cache.plan()
        assert {it[1] for it in items} == set(range(kv_hi - kv_lo))
    else:
        part = lpt_partition(ctx, world)[rank]
        q = synth.gen_rows(0, 0, part, [ctx[b] - 1 for b in part], Hq, D, "bf16")
        ks = [synth.gen_seq(1, 0, b, ctx[b], Hkv, D, "bf16") for b in part]
        vs = [synth.gen_seq(2, 0, b, ctx[b], Hkv, D, "bf16") for b in part]
        local = oa.decode_attention(q, ks, vs, "bf16", nthreads=1)
        got = [None] * world
        dist.all_gather_object(got, (part, local))
        full = np.zeros((B, Hq, D))
        for p, o in got:
            full[p] = o
        full = torch.from_numpy(full)
    if rank == 0:
        torch.save(full, result_path)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["head", "req"])
def test_sharded_equals_unsharded_gloo(tmp_path, mode):
    import torch

    from oracle import attention as oa
    oa.build()
    path = str(tmp_path / "full.pt")
    mp.spawn(_worker, args=(2, _free_port(), mode, path), nprocs=2, join=True)
    got = torch.load(path).numpy()
    B, Hq, Hkv, D = 6, 8, 4, 128
    ctx = [3, 40, 17, 100, 1, 64]
    q = synth.gen_rows(0, 0, range(B), [c - 1 for c in ctx], Hq, D, "bf16")
    ks = [synth.gen_seq(1, 0, b, c, Hkv, D, "bf16") for b, c in enumerate(ctx)]
    vs = [synth.gen_seq(2, 0, b, c, Hkv, D, "bf16") for b, c in enumerate(ctx)]
    ref = oa.decode_attention(q, ks, vs, "bf16", nthreads=1)
    assert np.array_equal(got, ref)
