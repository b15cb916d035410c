"""Fused all-gather epilogue on one GPU.

Two head-sharded "ranks" (two handles, each owning half of the KV heads and
their q-groups) decode the same batch and each writes its head slice straight
into BOTH full-width output buffers (standing in for the two ranks' symmetric,
peer-mapped buffers) via apex_decode_attention_ex.  Both buffers must end up
identical and equal to the unsharded result (and the oracle).  On an 8-GPU box
the destinations would be NVLink peer pointers; that path is not exercised here
(one GPU).
"""
import pytest

from helpers import check_close, gen_dev, make_cache, oracle_rows, to_f64

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype,hq,hkv,world", [("bf16", 32, 8, 2), ("bf16", 32, 8, 4), ("f16", 8, 8, 2)])
def test_head_sharded_epilogue_gather(cuda_lib, dtype, hq, hkv, world):
    import torch

    import synth
    from paper_2506_03296_b200.kvcache import torch_dtype
    ctx = [1, 300, 2000, 4096, 17]
    B = len(ctx)
    seqs = list(range(B))
    hkv_l, hq_l = hkv // world, hq // world
    full = [torch.full((B, hq, 128), float("nan"), dtype=torch_dtype(dtype), device="cuda") for _ in range(world)]
    ranks = []
    for r in range(world):
        c = make_cache(dtype, hq_l, hkv_l, sum(-(-x // 16) for x in ctx) + 4, max_seqs=B,
                       max_blocks_per_seq=max(-(-x // 16) for x in ctx) + 1)
        # prefill + step with this rank's slice of the global heads
        pre = {s: x - 1 for s, x in zip(seqs, ctx) if x > 1}
        c.alloc(list(pre), list(pre.values()))
        rb = [s for s in pre for _ in range(pre[s])]
        rp = [t for s in pre for t in range(pre[s])]
        from paper_2506_03296_b200.kvcache import synth_rows
        kk = torch.empty((len(rb), hkv_l, 128), dtype=torch_dtype(dtype), device="cuda")
        vv = torch.empty_like(kk)
        synth_rows(kk, dtype, 1, 0, torch.tensor(rb), torch.tensor(rp), head_offset=r * hkv_l)
        synth_rows(vv, dtype, 2, 0, torch.tensor(rb), torch.tensor(rp), head_offset=r * hkv_l)
        c.append(0, kk, vv)
        c.alloc(seqs, [1] * B)
        pos = torch.tensor([x - 1 for x in ctx])
        k1 = torch.empty((B, hkv_l, 128), dtype=torch_dtype(dtype), device="cuda")
        v1 = torch.empty_like(k1)
        q1 = torch.empty((B, hq_l, 128), dtype=torch_dtype(dtype), device="cuda")
        synth_rows(k1, dtype, 1, 0, torch.tensor(seqs), pos, head_offset=r * hkv_l)
        synth_rows(v1, dtype, 2, 0, torch.tensor(seqs), pos, head_offset=r * hkv_l)
        synth_rows(q1, dtype, 0, 0, torch.tensor(seqs), pos, head_offset=r * hq_l)
        c.append(0, k1, v1)
        c.decode_into(0, q1, full, head_offset=r * hq_l)     # every rank writes into every buffer
        ranks.append(c)
    torch.cuda.synchronize()
    for f in full[1:]:
        assert torch.equal(f, full[0])
    ref = oracle_rows(seqs, ctx, hq, hkv, dtype)
    check_close(to_f64(full[0], dtype), ref, dtype)


def _run_handle(dtype, hq_l, hkv_l, head_off_q, head_off_kv, ctx, req_ids, split):
    """One handle serving requests req_ids (generator ids) with a slice of the heads."""
    import torch

    from paper_2506_03296_b200.kvcache import synth_rows, torch_dtype
    B = len(ctx)
    c = make_cache(dtype, hq_l, hkv_l, sum(-(-x // 16) for x in ctx) + 4, max_seqs=B,
                   max_blocks_per_seq=max(-(-x // 16) for x in ctx) + 1)
    c.set_split(split)
    seqs = list(range(B))
    pre = {s: x - 1 for s, x in zip(seqs, ctx) if x > 1}
    tdt = torch_dtype(dtype)
    if pre:
        c.alloc(list(pre), list(pre.values()))
        rb = [req_ids[s] for s in pre for _ in range(pre[s])]
        rp = [t for s in pre for t in range(pre[s])]
        kk = torch.empty((len(rb), hkv_l, 128), dtype=tdt, device="cuda")
        vv = torch.empty_like(kk)
        synth_rows(kk, dtype, 1, 0, torch.tensor(rb), torch.tensor(rp), head_offset=head_off_kv)
        synth_rows(vv, dtype, 2, 0, torch.tensor(rb), torch.tensor(rp), head_offset=head_off_kv)
        c.append(0, kk, vv)
    c.alloc(seqs, [1] * B)
    pos, ids = torch.tensor([x - 1 for x in ctx]), torch.tensor(req_ids)
    k1 = torch.empty((B, hkv_l, 128), dtype=tdt, device="cuda")
    v1 = torch.empty_like(k1)
    q1 = torch.empty((B, hq_l, 128), dtype=tdt, device="cuda")
    synth_rows(k1, dtype, 1, 0, ids, pos, head_offset=head_off_kv)
    synth_rows(v1, dtype, 2, 0, ids, pos, head_offset=head_off_kv)
    synth_rows(q1, dtype, 0, 0, ids, pos, head_offset=head_off_q)
    c.append(0, k1, v1)
    out = c.decode(0, q1)
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("dtype,hq,hkv", [("bf16", 32, 8), ("f16", 8, 8)])
def test_sharded_bit_identical_to_unsharded(cuda_lib, dtype, hq, hkv):
    """SURVEY §4 dist_head_vs_1gpu / dist_req_vs_1gpu on one GPU: with the split chunk
    fixed, head-sharded and request-sharded outputs equal the unsharded output bit for bit."""
    import torch
    ctx = [1, 300, 2000, 4096, 17, 777]
    ids = list(range(len(ctx)))
    full = _run_handle(dtype, hq, hkv, 0, 0, ctx, ids, 256)
    world = 2
    for r in range(world):                                   # head sharding
        o = _run_handle(dtype, hq // world, hkv // world, r * hq // world, r * hkv // world, ctx, ids, 256)
        assert torch.equal(o, full[:, r * hq // world:(r + 1) * hq // world])
    from paper_2506_03296_b200.sharding import lpt_partition
    for part in lpt_partition(ctx, world):                   # request sharding
        o = _run_handle(dtype, hq, hkv, 0, 0, [ctx[i] for i in part], [ids[i] for i in part], 256)
        assert torch.equal(o, full[part])
