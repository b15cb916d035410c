"""Run one decode step for an arbitrary shape and compare with the oracle (debug aid).
    python tools/debug_case.py --dtype f16 --hq 32 --hkv 32 --batch 8 --ctx 4096 [--split 0]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch

    from helpers import check_close, decode_step, make_cache, oracle_rows, prefill, to_f64
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="f16")
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=32)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--ctx", type=int, default=4096)
    ap.add_argument("--split", type=int, default=0)
    a = ap.parse_args()
    ctx = [a.ctx] * a.batch
    cache = make_cache(a.dtype, a.hq, a.hkv, a.batch * (a.ctx // 16 + 2), max_seqs=a.batch,
                       max_blocks_per_seq=a.ctx // 16 + 2)
    if a.split:
        cache.set_split(a.split)
    seqs = list(range(a.batch))
    prefill(cache, seqs, ctx)
    out = decode_step(cache, seqs, ctx)
    torch.cuda.synchronize()
    items, nm = cache.plan()
    print("items", len(items), "merges", nm, "sizes", sorted({i[3] for i in items}))
    rows = list(range(min(64, a.batch * a.hq)))
    ref = oracle_rows(seqs, ctx, a.hq, a.hkv, a.dtype, rows=rows)
    print("err", check_close(to_f64(out, a.dtype).reshape(-1, 128)[rows], ref, a.dtype))


if __name__ == "__main__":
    main()
