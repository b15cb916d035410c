"""Maximum-size edge case: LLaMA-3.1's 128K-token context (131072 tokens, 8192
blocks per sequence), in both planner regimes, against the float64 oracle.

Latency regime: one 128K request next to a ctx-1 and a 5000-token request (one
launch, the 128K pairs split into many parts merged in-kernel by the last
arriver).  Bandwidth regime: 16 x 128K (guided split + merge kernel; the pool
is 2 GiB, byte offsets past 2^31).  Shapes: Hq 8 / Hkv 2 (a rank's slice of
LLaMA-3.1-8B under 4-way head sharding) so that the host oracle's regenerated
K/V stay small; sampled rows cover the first and last request.
"""
import pytest

from helpers import check_close, decode_step, make_cache, oracle_rows, prefill, to_f64

pytestmark = pytest.mark.gpu

MAXCTX = 131072


@pytest.mark.parametrize("ctx,launches", [([MAXCTX, 1, 5000], 1), ([MAXCTX] * 16, 2)])
def test_max_context(cuda_lib, ctx, launches):
    import torch
    dtype, hq, hkv = "bf16", 8, 2
    B = len(ctx)
    nb = sum(-(-c // 16) for c in ctx) + 16
    cache = make_cache(dtype, hq, hkv, nb, max_seqs=B, max_blocks_per_seq=MAXCTX // 16 + 1,
                       max_new_tokens=1 << 22)
    seqs = list(range(B))
    prefill(cache, seqs, ctx)
    out = to_f64(decode_step(cache, seqs, ctx), dtype)
    assert cache.decode_launches() == launches
    items, _ = cache.plan()
    assert max(nblk for (_, _, _, nblk, _, _) in items) < MAXCTX // 16      # the long pairs are split
    pick = [0, B - 1] if B > 3 else list(range(B))
    rows = [b * hq + h for b in pick for h in range(hq)]
    ref = oracle_rows(seqs, ctx, hq, hkv, dtype, rows=rows)
    check_close(out.reshape(-1, 128)[rows], ref, dtype)
    ln, blocks = cache.seq_info(0)
    assert ln == MAXCTX and len(blocks) == MAXCTX // 16
    del cache
    torch.cuda.empty_cache()
