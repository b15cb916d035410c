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


@pytest.mark.parametrize("dtype,hq,hkv,world", [("bf16", 32, 8, 2), ("bf16", 32, 8, 4), ("bf16", 32, 8, 8),
                                                ("f16", 8, 8, 2)])
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


def _rank_cache(dtype, hq, hkv, world, r, ctx, seqs, layers=1, stream=None):
    """A 'rank' of head sharding on this GPU: its kv-head slice prefilled for every
    layer, then one decode step allocated (append of the step's token done).  Returns
    (cache, q of the step per layer)."""
    import torch

    from paper_2506_03296_b200.kvcache import synth_rows, torch_dtype
    B = len(ctx)
    hkv_l, hq_l = hkv // world, hq // world
    tdt = torch_dtype(dtype)
    c = make_cache(dtype, hq_l, hkv_l, sum(-(-x // 16) for x in ctx) + 4, max_seqs=B,
                   max_blocks_per_seq=max(-(-x // 16) for x in ctx) + 1, layers=layers)
    pre = {s: x - 1 for s, x in zip(seqs, ctx) if x > 1}
    c.alloc(list(pre), list(pre.values()))
    rb = torch.tensor([s for s in pre for _ in range(pre[s])])
    rp = torch.tensor([t for s in pre for t in range(pre[s])])
    for l in range(layers):
        kk = torch.empty((len(rb), hkv_l, 128), dtype=tdt, device="cuda")
        vv = torch.empty_like(kk)
        synth_rows(kk, dtype, 1, l, rb, rp, head_offset=r * hkv_l)
        synth_rows(vv, dtype, 2, l, rb, rp, head_offset=r * hkv_l)
        c.append(l, kk, vv)
    c.alloc(seqs, [1] * B)
    pos = torch.tensor([x - 1 for x in ctx])
    qs = []
    for l in range(layers):
        k1 = torch.empty((B, hkv_l, 128), dtype=tdt, device="cuda")
        v1 = torch.empty_like(k1)
        q1 = torch.empty((B, hq_l, 128), dtype=tdt, device="cuda")
        synth_rows(k1, dtype, 1, l, torch.tensor(seqs), pos, head_offset=r * hkv_l)
        synth_rows(v1, dtype, 2, l, torch.tensor(seqs), pos, head_offset=r * hkv_l)
        synth_rows(q1, dtype, 0, l, torch.tensor(seqs), pos, head_offset=r * hq_l)
        c.append(l, k1, v1)
        qs.append(q1)
    return c, qs


@pytest.mark.parametrize("split", [0, 64])
def test_head_major_layout(cuda_lib, split):
    """a7 layout: each rank writes its heads head-major ([Hq/N][B][D], row stride D, head
    stride B*D), so the concatenation of the rank slices IS the gathered [Hq][B][D]
    (what all_gather_into_tensor produces) -- equal to the oracle, both planner regimes
    (split 64: bandwidth-style split + merge kernel; 0: automatic)."""
    import torch

    from paper_2506_03296_b200.kvcache import torch_dtype
    dtype, hq, hkv, world = "bf16", 32, 8, 2
    ctx = [1, 300, 2000, 4096, 17]
    seqs = list(range(len(ctx)))
    slices = []
    for r in range(world):
        c, (q,) = _rank_cache(dtype, hq, hkv, world, r, ctx, seqs)
        c.set_split(split)
        c.alloc(seqs, [0] * len(seqs))                  # re-plan with the split (no new token)
        local = torch.full((hq // world, len(ctx), 128), float("nan"), dtype=torch_dtype(dtype), device="cuda")
        c.decode_into(0, q, [local], layout="hbd")
        slices.append(local)
    torch.cuda.synchronize()
    full = torch.cat(slices, 0)                         # [Hq][B][D]
    ref = oracle_rows(seqs, ctx, hq, hkv, dtype)        # [B][Hq][D]
    check_close(to_f64(full.permute(1, 0, 2), dtype), ref, dtype)


def test_decode_into_rejects_bad_outputs(cuda_lib):
    import torch
    c, (q,) = _rank_cache("bf16", 32, 8, 1, 0, [40, 50], [0, 1])
    ok = torch.empty((2, 32, 128), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError):
        c.decode_into(0, q, [ok, torch.empty((2, 16, 128), dtype=torch.bfloat16, device="cuda")])
    with pytest.raises(ValueError):
        c.decode_into(0, q, [ok], head_offset=8)        # 8 + 32 heads > 32
    with pytest.raises(ValueError):
        c.decode_into(0, q, [torch.empty((32, 2, 128), dtype=torch.bfloat16, device="cuda")], layout="bhd")
    from paper_2506_03296_b200 import apex as A
    with pytest.raises(A.ApexError):                    # overlapping strides refused by the ABI
        A.apex_decode_attention_ex(c.handle, 0, q.data_ptr(), [ok.data_ptr()], 128, 128, 0, 0.1)


@pytest.mark.parametrize("split", [0, 64])
def test_signalled_gather_in_kernel_flags(cuda_lib, split):
    """f3 completion flags: two head-sharded 'ranks' on one GPU write their slices into
    both ranks' [Hq][B][D] buffers and post their epoch into both ready arrays from the
    kernel's last CTA (fused merge: decode kernel; split 64: merge kernel).  A reader
    stream that waits on the flags BEFORE the writers are even launched must see the
    complete rows; buffers equal each other and the oracle; two epochs with the
    write-after-read guard (free flags) posted by the readers."""
    import torch

    from paper_2506_03296_b200.kvcache import torch_dtype
    from paper_2506_03296_b200.sharding import SignalledGather
    dtype, hq, hkv, world = "bf16", 32, 8, 2
    ctx = [1, 300, 2000, 4096, 17]
    seqs, B = list(range(len(ctx))), len(ctx)
    caches, qs = [], []
    for r in range(world):
        c, (q,) = _rank_cache(dtype, hq, hkv, world, r, ctx, seqs)
        c.set_split(split)
        c.alloc(seqs, [0] * B)
        caches.append(c)
        qs.append(q)
    bufs = [torch.full((hq, B, 128), float("nan"), dtype=torch_dtype(dtype), device="cuda") for _ in range(world)]
    sig = [torch.zeros((2, world), dtype=torch.int32, device="cuda") for _ in range(world)]   # [ready; free]
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    ptr = lambda t, off=0: t.data_ptr() + off
    gathers = [SignalledGather(r, world, [[ptr(b) for b in bufs]], [[ptr(s) for s in sig]],
                               [[ptr(s, 4 * world) for s in sig]]) for r in range(world)]
    [b.clone() for b in bufs]                           # load the copy kernel before anything spins: with
    torch.cuda.synchronize()                            # lazy loading its first launch would block the host
    reader = torch.cuda.Stream()                        # behind the reader's spinning wait
    writer = torch.cuda.Stream()
    ref = oracle_rows(seqs, ctx, hq, hkv, dtype)
    for epoch in (1, 2):
        snaps = []
        with torch.cuda.stream(reader):                 # queued first: spins until the flags land
            for r in range(world):
                gathers[r].wait_ready(0, epoch, reader.cuda_stream, status.data_ptr())
            snaps = [b.clone() for b in bufs]
            for r in range(world):
                gathers[r].release(0, epoch, reader.cuda_stream)
        with torch.cuda.stream(writer):
            if epoch == 2:                              # epoch-1 readers released the buffers
                for b in bufs:
                    b.fill_(float("nan"))
            for r in range(world):
                gathers[r].decode(caches[r], 0, qs[r], epoch, hq, status.data_ptr())
        torch.cuda.synchronize()
        assert int(status.item()) == 0, "a flag wait timed out"
        for s in sig:
            assert s.tolist() == [[epoch] * world, [epoch] * world]
        for snap in snaps:
            assert torch.equal(snap, snaps[0])
            check_close(to_f64(snap.permute(1, 0, 2), dtype), ref, dtype)


def test_signal_wait_timeout_does_not_hang(cuda_lib):
    import torch

    from paper_2506_03296_b200 import apex as A
    flags = torch.zeros(4, dtype=torch.int32, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    A.apex_signal_wait(flags.data_ptr(), 4, 1, 2_000_000, status.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert int(status.item()) == 1
    A.apex_signal_post([flags.data_ptr(), flags.data_ptr() + 8], 1, 7, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert flags.tolist() == [0, 7, 0, 7]
    status.zero_()
    A.apex_signal_wait(flags.data_ptr() + 4, 1, 7, 2_000_000_000, status.data_ptr(),
                       torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
