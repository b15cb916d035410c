"""Per-CTA timeline of one decode call (tuning aid; needs a libapex built with -DAPEX_TRACE).

    APEX_LIB=ab/trace.so python tools/trace_probe.py --shape bf16,32,8,1,16384
Events (globaltimer ns, relative to the first CTA start): 0 CTA start, 1 after griddepcontrol.wait,
2 first item published, 3 first block-table chunk loaded, 4 producer done, 5 first tile landed
(consumer 0), 6 consumer 0 done with item 0 tiles, 7 item-0 warp states merged, 8 item-0 output/partial
stored, 13 arrival fence done (thread 32), 9 fused-merge arrival decided, 10 fused merge done, 11 CTA consumers exit, 12 CTA exit after
the completion signal; slot 14 = merge pair + 1 of item 0, 15 = 1 if this CTA merged that pair.
--dump writes the per-CTA matrix and a critical-path summary per merged pair.
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch

    from helpers import gen_dev, make_cache, prefill
    from paper_2506_03296_b200 import apex as A
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="bf16,32,8,1,16384")
    ap.add_argument("--no-flush", action="store_true", help="keep L2 warm between calls")
    ap.add_argument("--flush", choices=["read", "write"], default="read")
    ap.add_argument("--dump", default="", help="write the raw per-CTA trace + pair analysis (JSON) here")
    a = ap.parse_args()
    d, *n = a.shape.split(",")
    dtype, (hq, hkv, batch, ctx) = d, [int(x) for x in n]
    L = A.lib()
    L.apex_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
    flush = torch.zeros(512 << 20, dtype=torch.uint8, device="cuda")
    sink = torch.zeros((), dtype=torch.int64, device="cuda")
    cache = make_cache(dtype, hq, hkv, batch * (-(-(ctx + 1) // 16)) + 8, max_seqs=batch,
                       max_blocks_per_seq=-(-(ctx + 1) // 16) + 1, max_new_tokens=1 << 22)
    seqs = list(range(batch))
    prefill(cache, seqs, [ctx] * batch)
    cache.alloc(seqs, [1] * batch)
    k = gen_dev(cache, 1, 0, seqs, [ctx] * batch, hkv)
    cache.append(0, k, k)
    q = gen_dev(cache, 0, 0, seqs, [ctx] * batch, hq)
    out = torch.empty_like(q)
    for r in range(4):
        if not a.no_flush:
            if a.flush == "write":
                flush.fill_(r)
            else:
                sink.copy_(flush.view(torch.int64).sum())
        L.apex_debug_trace_clear()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cache.decode(0, q, out=out)
        e1.record()
        torch.cuda.synchronize()
    buf = np.zeros((1024, 16), dtype=np.uint64)
    L.apex_debug_trace(buf.ctypes.data, 1024)
    P = len(cache.plan_ranges()) - 1
    t = buf[:P].astype(np.int64)
    t0 = t[:, 0][t[:, 0] > 0].min()
    res = {"shape": a.shape, "event_us": e0.elapsed_time(e1) * 1e3, "ctas": P, "items": len(cache.plan()[0])}
    for ev in range(14):
        v = t[:, ev]
        v = v[v > 0]
        if len(v):
            rel = (v - t0) / 1e3
            res[f"ev{ev}"] = {"n": int(len(v)), "min": round(float(rel.min()), 2), "p50": round(float(np.median(rel)), 2),
                              "max": round(float(rel.max()), 2)}
    # critical path of the fused merges: per pair, the last partial stored (ev8 max over its
    # splits), the merger's arrival decision (ev9) and merge end (ev10)
    rel = lambda x: (int(x) - int(t0)) / 1e3
    pairs = {}
    for c in range(P):
        mg = int(t[c, 14])
        if mg > 0 and t[c, 8] > 0:
            d = pairs.setdefault(mg - 1, {"parts": 0, "last_stored": 0.0})
            d["parts"] += 1
            d["last_stored"] = max(d["last_stored"], rel(t[c, 8]))
            if t[c, 15] == 1:
                d.update(merger=c, arrive=rel(t[c, 9]), merged=rel(t[c, 10]), fenced=rel(t[c, 13]),
                         stored=rel(t[c, 8]))
    if pairs:
        m = [d for d in pairs.values() if "merger" in d]
        res["pairs"] = len(pairs)
        res["merge_us_p50"] = round(float(np.median([d["merged"] - d["arrive"] for d in m])), 2) if m else None
        res["fence_us_p50"] = round(float(np.median([d["fenced"] - d["stored"] for d in m])), 2) if m else None
        res["atomic_us_p50"] = round(float(np.median([d["arrive"] - d["fenced"] for d in m])), 2) if m else None
        res["arrive_after_last_store_p50"] = round(float(np.median([d["arrive"] - d["last_stored"] for d in m])), 2) if m else None
        res["last_stored_max"] = round(max(d["last_stored"] for d in pairs.values()), 2)
        res["merged_max"] = round(max(d["merged"] for d in m), 2) if m else None
    ends = np.maximum(t[:, 11], t[:, 12])
    ends = ends[ends > 0]
    if len(ends):
        res["kernel_span_us"] = round(rel(ends.max()), 2)
    print(json.dumps(res))
    if a.dump:
        with open(a.dump, "w") as f:
            json.dump({"summary": res, "t0": int(t0), "trace": t.tolist(), "pairs": pairs}, f)


if __name__ == "__main__":
    main()
