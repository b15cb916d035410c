"""Device time of one decode step's pieces in the latency regime, L2 flushed (read) first.

    APEX_LIB=... python tools/alloc_probe.py [--reps 25]
Per shape: median us between CUDA events around apex_kv_alloc (metadata upload + table
deltas), around the fused append+decode call, and around the whole step (alloc + call).
The host has the flush's ~100 us to enqueue everything, so the intervals are GPU time.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

SHAPES = [("f32", 32, 32, 1, 512), ("bf16", 32, 8, 1, 4096), ("bf16", 32, 8, 64, 1024), ("bf16", 32, 8, 256, 512)]


def main():
    import torch

    from helpers import gen_dev, make_cache, prefill
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=25)
    a = ap.parse_args()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    sink = torch.zeros((), dtype=torch.int64, device="cuda")
    for dt, hq, hkv, B, ctx0 in SHAPES:
        steps = a.reps + 3
        ctx = [ctx0] * B
        cache = make_cache(dt, hq, hkv, B * (-(-(ctx0 + steps) // 16)) + 16, max_seqs=B,
                           max_blocks_per_seq=-(-(ctx0 + steps) // 16) + 1)
        seqs = list(range(B))
        prefill(cache, seqs, ctx)
        t_alloc, t_call, t_step = [], [], []
        for s in range(steps):
            pos = [c - 1 + s for c in ctx]
            q = gen_dev(cache, 0, 0, seqs, pos, hq)
            k = gen_dev(cache, 1, 0, seqs, pos, hkv)
            v = gen_dev(cache, 2, 0, seqs, pos, hkv)
            sink.copy_(flush.view(torch.int64).sum())
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record()
            cache.alloc(seqs, [1] * B)
            e[1].record()
            cache.decode_append(0, q, k, v)
            e[2].record()
            torch.cuda.synchronize()
            if s >= 3:
                t_alloc.append(e[0].elapsed_time(e[1]) * 1e3)
                t_call.append(e[1].elapsed_time(e[2]) * 1e3)
                t_step.append(e[0].elapsed_time(e[2]) * 1e3)
        print(json.dumps({"dtype": dt, "hq": hq, "hkv": hkv, "batch": B, "ctx": ctx0,
                          "lib": os.path.basename(os.environ.get("APEX_LIB", "libapex.so")),
                          "alloc_us": round(statistics.median(t_alloc), 2),
                          "call_us": round(statistics.median(t_call), 2),
                          "step_us": round(statistics.median(t_step), 2),
                          "launches": cache.decode_launches()}), flush=True)
        cache.close()
        del cache
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
