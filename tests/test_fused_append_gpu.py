"""apex_decode_attention_append: append + decode in one launch.

For pure decode steps the fused call must leave the pools byte-identical to
apex_kv_append and return outputs bit-identical to apex_kv_append +
apex_decode_attention, across block boundaries, in both planner regimes, and
within tolerance of the float64 oracle."""
import numpy as np
import pytest

from helpers import check_close, gen_dev, make_cache, oracle_rows, prefill, to_f64

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype,hq,hkv,ctx,launches", [("bf16", 32, 8, [1, 15, 16, 17, 300, 2000], 1),
                                                       ("f16", 32, 32, [5, 31, 32, 1000], 1),
                                                       ("f32", 8, 8, [2, 16, 100], 1),
                                                       ("f16", 16, 2, [1, 33, 4096], 1),
                                                       # latency regime near its edge: T = 82240 <= 512 * 296
                                                       ("bf16", 32, 8, [4096] * 40, 1),
                                                       # bandwidth regime: T = 40 * 513 * 8 = 164160 > 512 * 296
                                                       # (append kernel + decode kernel + merge kernel)
                                                       ("bf16", 32, 8, [8192] * 40, 2)])
def test_fused_append_matches_two_calls(cuda_lib, dtype, hq, hkv, ctx, launches):
    import torch
    B, steps = len(ctx), 18                                      # crosses a 16-token block boundary
    nb = sum(-(-(c + steps) // 16) for c in ctx) + 8
    mb = -(-(max(ctx) + steps) // 16) + 1
    fused = make_cache(dtype, hq, hkv, nb, max_seqs=B, max_blocks_per_seq=mb)
    ref = make_cache(dtype, hq, hkv, nb, max_seqs=B, max_blocks_per_seq=mb)
    seqs = list(range(B))
    for c in (fused, ref):
        c.kv_pools[0].zero_()                                     # unwritten slots compare equal
        prefill(c, seqs, ctx)
    for s in range(steps):
        cur = [c + s for c in ctx]
        pos = [c - 1 for c in cur]
        for c in (fused, ref):
            c.alloc(seqs, [1] * B)
        q = gen_dev(fused, 0, 0, seqs, pos, hq)
        k = gen_dev(fused, 1, 0, seqs, pos, hkv)
        v = gen_dev(fused, 2, 0, seqs, pos, hkv)
        assert fused.decode_launches() == launches, "planner regime of the case"
        out_f = fused.decode_append(0, q, k, v)
        ref.append(0, k, v)
        out_r = ref.decode(0, q)
        torch.cuda.synchronize()
        assert torch.equal(out_f, out_r), f"fused != two calls at step {s}"
    assert torch.equal(fused.kv_pools[0], ref.kv_pools[0])      # same allocator -> same layout, same bytes
    rows = list(range(0, B * hq, max(1, B * hq // 48)))
    check_close(to_f64(out_f, dtype).reshape(-1, 128)[rows], oracle_rows(seqs, cur, hq, hkv, dtype, rows=rows), dtype)


def test_fused_append_rejects_multi_token_steps(cuda_lib):
    from paper_2506_03296_b200 import apex as A
    c = make_cache("bf16", 32, 8, 64, max_seqs=4, max_blocks_per_seq=16)
    prefill(c, [0, 1], [40, 10])
    c.alloc([0, 1], [1, 2])                                     # seq 1 gets two tokens
    q = gen_dev(c, 0, 0, [0, 1], [40, 11], 32)
    k = gen_dev(c, 1, 0, [0, 1], [40, 11], 8)
    with pytest.raises(A.ApexError) as e:
        c.decode_append(0, q, k, k)
    assert e.value.code == "EINVAL"
