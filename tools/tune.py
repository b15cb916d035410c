"""Decode-only timing sweep over planner settings on one physical layer (tuning aid).

    python tools/tune.py --config c3 [--chunks 0,512,1024,2048] [--reps 30]

Builds the config's cache once (one physical layer), appends one decode step,
then times apex_decode_attention back to back (CUDA events, median) for each
split chunk (0 = automatic planner).  Prints GB/s against the algorithmic bytes.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import numpy as np
    import torch

    from helpers import gen_dev, make_cache, prefill
    from synth import WORKLOADS
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--chunks", default="0,256,512,1024,2048,4096,8192,16384")
    ap.add_argument("--grids", default="0")
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--layers", type=int, default=1, help="physical layers; calls rotate over them")
    ap.add_argument("--scheds", default="", help="comma list of apex_kv_set_sched values (-1 dynamic, "
                                                 "0..1000 stream-K dynamic permille); empty = library default")
    a = ap.parse_args()
    w = WORKLOADS[a.config]
    ctx = [int(c) for c in w.contexts()]
    B = len(ctx)
    mult = int(os.environ.get("APEX_TUNE_BLOCK_MULT", "1"))     # >1: spare pool rows for layout experiments
    cache = make_cache(w.dtype, w.num_q_heads, w.num_kv_heads, mult * (sum(-(-(c + 1) // 16) for c in ctx) + 16),
                       max_seqs=B, max_blocks_per_seq=-(-(max(ctx) + 1) // 16) + 1, max_new_tokens=1 << 22,
                       layers=a.layers)
    seqs = list(range(B))
    prefill(cache, seqs, ctx)            # layer 0 holds data; the other layers' bytes are streamed as they are
    es = 4 if w.dtype == "f32" else 2
    nbytes = sum(c * w.num_kv_heads * 128 * 2 * es for c in ctx) + 2 * B * w.num_q_heads * 128 * es
    res = []
    # a sched entry "-2:8/800/900/950" sets the guided planner's constants (apex_kv_set_planner)
    scheds = a.scheds.split(",") if a.scheds else [None]
    for grid, chunk, sched in [(g, c, s) for g in [int(x) for x in a.grids.split(",")]
                               for c in [int(x) for x in a.chunks.split(",")] for s in scheds]:
        if True:
            cache.set_grid(grid)
            cache.set_split(chunk)
            if sched is not None:
                sv, _, gp = sched.partition(":")
                if gp:
                    div, p1, p2, p3 = [int(x) for x in gp.split("/")]
                    cache.set_planner(512, div, (p1, p2, p3))
                cache.set_sched(int(sv))
            try:
                cache.alloc(seqs, [0] * B)
            except Exception as e:          # chunk too small for the workspace
                print(f"grid {grid} chunk {chunk}: {e}")
                continue
            q = gen_dev(cache, 0, 0, seqs, [c - 1 for c in ctx], w.num_q_heads)
            out = torch.empty_like(q)
            for li in range(max(3, a.layers)):
                cache.decode(li % a.layers, q, out=out)
            ts = []
            for r in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                cache.decode(r % a.layers, q, out=out)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            items, merges = cache.plan()
            med = statistics.median(ts)
            r = dict(grid=grid, chunk=chunk, sched=sched, items=len(items), merges=merges, us_med=med, us_min=min(ts),
                     gbs=nbytes / med / 1e3)
            res.append(r)
            print(json.dumps(r), flush=True)
    print(json.dumps({"config": a.config, "bytes": nbytes, "results": res}))


if __name__ == "__main__":
    main()
