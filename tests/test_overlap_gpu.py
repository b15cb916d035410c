"""f4: the Asynchronous-Overlap analogue -- DeferredLane runs the
attention of an offloaded subset of requests on its own stream and cache while the
main stream does other work (a GEMM standing in for the linear layers); the layer's
result is collected only when it is ready, and a not-yet-ready result is reported
without stalling the caller (PAPER.md P:214-216 deferred synchronization, P:311
non-stalling re-check).  Results vs the float64 oracle."""
import time

import pytest

from helpers import check_close, gen_dev, make_cache, oracle_rows, prefill, to_f64

pytestmark = pytest.mark.gpu


def test_deferred_lane_parity_and_non_stalling(cuda_lib):
    import torch

    from paper_2506_03296_b200 import apex as A
    from paper_2506_03296_b200.overlap import DeferredLane
    dtype, hq, hkv, L = "bf16", 32, 8, 2
    ctx = [300, 2000, 17, 4096]
    seqs = list(range(len(ctx)))
    cache = make_cache(dtype, hq, hkv, sum(-(-c // 16) for c in ctx) + 8, max_seqs=len(ctx),
                       max_blocks_per_seq=max(-(-c // 16) for c in ctx) + 2, layers=L)
    prefill(cache, seqs, ctx, layer=list(range(L)))
    lane = DeferredLane(cache, L)
    pos = [c - 1 for c in ctx]
    qs = [gen_dev(cache, 0, l, seqs, pos, hq) for l in range(L)]
    ks = [gen_dev(cache, 1, l, seqs, pos, hkv) for l in range(L)]
    vs = [gen_dev(cache, 2, l, seqs, pos, hkv) for l in range(L)]
    a = torch.randn(2048, 2048, device="cuda", dtype=torch.bfloat16)
    # load every kernel the main stream launches below before anything spins: with CUDA
    # lazy loading the first launch of a kernel can block the host behind the spinning
    # gate until its timeout, after which the lane completes early
    ((a @ a) * 0.01).sum().item()
    gate = torch.zeros(1, dtype=torch.int32, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    lane.alloc(seqs, [1] * len(ctx))
    # hold the lane behind a gate so its layer-0 result cannot be ready yet
    A.apex_signal_wait(gate.data_ptr(), 1, 1, 20_000_000_000, status.data_ptr(), lane.stream.cuda_stream)
    for l in range(L):
        lane.launch(l, qs[l], ks[l], vs[l])
    y = a
    for _ in range(8):                           # the main stream's own work meanwhile
        y = (y @ a) * 0.01
    early = lane.collect(0)
    assert int(status.item()) == 0, "the gate timed out: the host blocked behind the spinning wait"
    assert early is None and not lane.ready(1)   # not ready: reported, no stall
    A.apex_signal_post([gate.data_ptr()], 0, 1, torch.cuda.current_stream().cuda_stream)
    t0 = time.time()
    outs = [None] * L
    while any(o is None for o in outs):          # re-check "next iteration" until ready
        for l in range(L):
            if outs[l] is None:
                outs[l] = lane.collect(l)
        assert time.time() - t0 < 20, "lane never completed"
        time.sleep(0.001)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    for l in range(L):
        check_close(to_f64(outs[l], dtype), oracle_rows(seqs, ctx, hq, hkv, dtype, layer=l), dtype)
    assert lane.collect(0) is None               # collected once
