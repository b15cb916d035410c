"""Per-CTA timeline of one decode call (tuning aid; needs a libapex built with -DAPEX_TRACE).

    APEX_LIB=ab/trace.so python tools/trace_probe.py --shape bf16,32,8,1,16384
Events (globaltimer ns, relative to the first CTA start): 0 CTA start, 1 after griddepcontrol.wait,
2 first item published, 3 first block-table chunk loaded, 4 producer done, 5 first tile landed
(consumer 0), 6 consumer 0 done with item 0 tiles, 7 item-0 warp states merged, 8 item-0 output/partial
stored, 9 fused-merge arrival decided, 10 fused merge done, 11 CTA consumers exit.
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
    a = ap.parse_args()
    d, *n = a.shape.split(",")
    dtype, (hq, hkv, batch, ctx) = d, [int(x) for x in n]
    L = A.lib()
    L.apex_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
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
            flush.fill_(r)
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
    for ev in range(16):
        v = t[:, ev]
        v = v[v > 0]
        if len(v):
            rel = (v - t0) / 1e3
            res[f"ev{ev}"] = {"n": int(len(v)), "min": round(float(rel.min()), 2), "p50": round(float(np.median(rel)), 2),
                              "max": round(float(rel.max()), 2)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
