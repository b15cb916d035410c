"""CUDA-graph serving mode: the per-layer launches (apex_kv_append +
apex_decode_attention) are captured once and replayed every step; only
apex_kv_alloc (host planner + metadata upload) runs outside the graph.

Valid because every launch parameter is step-invariant (counts come from the
device step header, fixed grids, fixed upload offsets) -- see apex_internal.h.
Checked bit-for-bit against eager execution and against the float64 oracle
across steps that cross block boundaries and change the split plan.
"""
import numpy as np
import pytest

from helpers import check_close, gen_dev, make_cache, oracle_rows, prefill, to_f64

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype,hq,hkv,ctx", [("bf16", 32, 8, [5, 700, 2000, 31]), ("f16", 8, 8, [100, 3000]),
                                              ("f32", 4, 4, [15, 64, 999]),
                                              ("bf16", 32, 8, [8192] * 40)])   # bandwidth regime + merges
@pytest.mark.parametrize("fused_append", [False, True])
def test_graph_replay_matches_eager_and_oracle(cuda_lib, dtype, hq, hkv, ctx, fused_append):
    import torch
    B = len(ctx)
    steps = 18                                          # crosses a 16-token block boundary
    nb = sum(-(-(c + steps) // 16) for c in ctx) + 8
    mb = -(-(max(ctx) + steps) // 16) + 1
    graph_c = make_cache(dtype, hq, hkv, nb, max_seqs=B, max_blocks_per_seq=mb)
    eager_c = make_cache(dtype, hq, hkv, nb, max_seqs=B, max_blocks_per_seq=mb)
    seqs = list(range(B))
    for c in (graph_c, eager_c):
        prefill(c, seqs, ctx)
    D = 128
    from paper_2506_03296_b200.kvcache import torch_dtype
    tdt = torch_dtype(dtype)
    q_buf = torch.empty((B, hq, D), dtype=tdt, device="cuda")
    k_buf = torch.empty((B, hkv, D), dtype=tdt, device="cuda")
    v_buf = torch.empty((B, hkv, D), dtype=tdt, device="cuda")
    out_buf = torch.empty((B, hq, D), dtype=tdt, device="cuda")
    graph = None
    for s in range(steps):
        cur = [c + s for c in ctx]
        pos = [c - 1 for c in cur]
        for c in (graph_c, eager_c):
            c.alloc(seqs, [1] * B)
        q_buf.copy_(gen_dev(graph_c, 0, 0, seqs, pos, hq))
        k_buf.copy_(gen_dev(graph_c, 1, 0, seqs, pos, hkv))
        v_buf.copy_(gen_dev(graph_c, 2, 0, seqs, pos, hkv))
        if graph is None:
            stream = torch.cuda.Stream()
            stream.wait_stream(torch.cuda.current_stream())
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.stream(stream):
                with torch.cuda.graph(graph, stream=stream):
                    if fused_append:
                        graph_c.decode_append(0, q_buf, k_buf, v_buf, out=out_buf)
                    else:
                        graph_c.append(0, k_buf, v_buf)
                        graph_c.decode(0, q_buf, out=out_buf)
            torch.cuda.current_stream().wait_stream(stream)
        graph.replay()
        eager_c.append(0, k_buf, v_buf)
        ref_out = eager_c.decode(0, q_buf)
        torch.cuda.synchronize()
        assert torch.equal(out_buf, ref_out), f"graph != eager at step {s}"
    ref = oracle_rows(seqs, cur, hq, hkv, dtype, rows=list(range(0, B * hq, max(1, B * hq // 32))))
    got = to_f64(out_buf, dtype).reshape(-1, D)[list(range(0, B * hq, max(1, B * hq // 32)))]
    check_close(got, ref, dtype)
