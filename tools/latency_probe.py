"""Decode-call latency in the latency regime (few tiles per CTA), L2 flushed before every call.

    python tools/latency_probe.py [--reps 15]
Prints one JSON line per shape: dtype, heads, batch, ctx, median us per apex_decode_attention
(CUDA events around the call only; a 512 MiB write before each call evicts the KV from L2),
work items, decode launches and achieved GB/s against the algorithmic KV bytes.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

SHAPES = [("f32", 32, 32, 1, 512), ("bf16", 32, 8, 1, 512), ("bf16", 32, 8, 1, 4096), ("bf16", 32, 8, 1, 16384),
          ("bf16", 32, 8, 1, 65536), ("bf16", 32, 8, 4, 4096), ("bf16", 32, 8, 16, 2048), ("bf16", 32, 8, 64, 1024),
          ("f16", 32, 32, 8, 1024), ("f16", 32, 32, 1, 4096)]


def main():
    import torch

    from helpers import gen_dev, make_cache, prefill
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--shape", default="", help="dtype,hq,hkv,batch,ctx (default: the built-in list)")
    ap.add_argument("--sched", type=int, default=None, help="apex_kv_set_sched value")
    ap.add_argument("--lat-tiles", type=int, default=512, help="apex_kv_set_planner latency_tiles_per_cta")
    ap.add_argument("--graph", action="store_true", help="time a CUDA-graph replay of the call")
    ap.add_argument("--split", type=int, default=0, help="apex_kv_set_split chunk in tokens (0: planner)")
    ap.add_argument("--flush", choices=["read", "write"], default="read",
                    help="L2 flush before each call: read a 512 MiB buffer (L2 left clean) or write it (L2 left "
                         "full of dirty lines whose write-back competes with the decode's reads)")
    a = ap.parse_args()
    shapes = SHAPES
    if a.shape:
        d, *n = a.shape.split(",")
        shapes = [(d, *[int(x) for x in n])]
    flush = torch.zeros(512 << 20, dtype=torch.uint8, device="cuda")
    flush_sink = torch.zeros((), dtype=torch.int64, device="cuda")
    for dtype, hq, hkv, batch, ctx in shapes:
        cache = make_cache(dtype, hq, hkv, batch * (-(-(ctx + 1) // 16)) + 8, max_seqs=batch,
                           max_blocks_per_seq=-(-(ctx + 1) // 16) + 1, max_new_tokens=1 << 22)
        seqs = list(range(batch))
        prefill(cache, seqs, [ctx] * batch)
        cache.set_planner(a.lat_tiles)
        if a.sched is not None:
            cache.set_sched(a.sched)
        if a.split:
            cache.set_split(a.split)
        cache.alloc(seqs, [1] * batch)
        k = gen_dev(cache, 1, 0, seqs, [ctx] * batch, hkv)
        cache.append(0, k, k)
        q = gen_dev(cache, 0, 0, seqs, [ctx] * batch, hq)
        out = torch.empty_like(q)
        times = []
        graph = None
        if a.graph:
            cache.decode(0, q, out=out)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                cache.decode(0, q, out=out)
        for r in range(a.reps + 3):
            if a.flush == "write":
                flush.fill_(r & 0xff)
            else:
                flush_sink.copy_(flush.view(torch.int64).sum())
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if graph is not None:
                graph.replay()
            else:
                cache.decode(0, q, out=out)
            e1.record()
            torch.cuda.synchronize()
            if r >= 3:
                times.append(e0.elapsed_time(e1) * 1e3)
        es = 4 if dtype == "f32" else 2
        kv = batch * (ctx + 1) * hkv * 128 * 2 * es
        us = statistics.median(times)
        print(json.dumps({"dtype": dtype, "hq": hq, "hkv": hkv, "batch": batch, "ctx": ctx + 1, "us": round(us, 2),
                          "us_min": round(min(times), 2), "items": len(cache.plan()[0]),
                          "launches": cache.decode_launches(), "gbs": round(kv / us / 1e3, 1),
                          "sched": a.sched, "lat_tiles": a.lat_tiles, "split": a.split, "graph": a.graph,
                          "flush": a.flush}), flush=True)
        cache.close()
        del cache
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
