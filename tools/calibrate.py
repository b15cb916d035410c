"""Calibrate apex_predict_time on this B200 (the APEX offline profiler, §3.1).

    python tools/calibrate.py [--out profiles/cost_table_b200.json] [--dtype bf16 --hq 32 --hkv 8]

Measures the device time of one apex_decode_attention layer-call (decode kernel
+ LSE merge) on a (batch, total kv tokens) grid with uniform contexts, L2
flushed before every timed launch (a real model's next layer reads different
KV), median of --reps launches.  Then measures held-out off-grid points and
reports apex_predict_time's relative error against them (this accuracy is
"parity unpinned" by the paper).  Output: the table in SPEC.md's
profile spirit plus the held-out report.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

# covers the benched operating points: C3 (128, 1M), C4 (256, 4.5M), C5 (1024, 16.8M)
BATCH = [1, 4, 16, 64, 256, 1024]
KV_TOTAL = [1 << 14, 1 << 16, 1 << 18, 1 << 20, 1 << 22, 1 << 24]


def measure(dtype, hq, hkv, batch, total, reps, flush):
    import torch

    from helpers import gen_dev, make_cache, prefill
    ctx = max(1, total // batch)
    cache = make_cache(dtype, hq, hkv, batch * (-(-(ctx + 1) // 16)) + 8, max_seqs=batch,
                       max_blocks_per_seq=-(-(ctx + 1) // 16) + 1, max_new_tokens=1 << 22)
    seqs = list(range(batch))
    # very long single contexts are grown 1M tokens at a time (bounded append size)
    prefill(cache, seqs, [ctx] * batch, interleave=(1 << 20) if ctx > (1 << 21) else 0)
    cache.alloc(seqs, [1] * batch)
    k = gen_dev(cache, 1, 0, seqs, [ctx - 1] * batch, hkv)
    cache.append(0, k, k)
    q = gen_dev(cache, 0, 0, seqs, [ctx - 1] * batch, hq)
    out = torch.empty_like(q)
    times = []
    for r in range(reps + 2):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        cache.decode(0, q, out=out)
        b.record()
        torch.cuda.synchronize()
        if r >= 2:
            times.append(a.elapsed_time(b) * 1e3)
    cache.close()
    del cache
    torch.cuda.empty_cache()
    return statistics.median(times), batch * ctx


def main():
    import random

    import torch

    from paper_2506_03296_b200 import apex as A
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--heldout", type=int, default=16)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "cost_table_b200.json"))
    a = ap.parse_args()
    flush = torch.empty(512 * 2 ** 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2
    t0 = time.time()
    us = [[0.0] * len(KV_TOTAL) for _ in BATCH]
    for i, b in enumerate(BATCH):
        for j, t in enumerate(KV_TOTAL):
            us[i][j], _ = measure(a.dtype, a.hq, a.hkv, b, t, a.reps, flush)
            print(f"batch {b:4d} kv {t:9d}: {us[i][j]:10.2f} us", flush=True)
    h = A.apex_cost_create(BATCH, KV_TOTAL, us)
    rnd = random.Random(0)
    held = []
    for _ in range(a.heldout):
        b = rnd.randint(BATCH[0], BATCH[-1])
        t = int(2 ** rnd.uniform(14, 24))
        t = max(t, b * 16)
        m, t_real = measure(a.dtype, a.hq, a.hkv, b, t, a.reps, flush)
        p = A.apex_predict_time(h, b, t_real)
        held.append({"batch": b, "kv_tokens": t_real, "measured_us": m, "predicted_us": p, "rel_err": (p - m) / m})
        print(f"held-out batch {b} kv {t_real}: measured {m:.1f} predicted {p:.1f} us", flush=True)
    errs = [abs(x["rel_err"]) for x in held]
    doc = {"what": "per-layer-call apex_decode_attention device time (decode + LSE merge), L2 flushed, median",
           "paper": "offline profiler + performance model, PAPER.md P:153, P:163-169; SPEC.md S:49-57, S:100",
           "device": torch.cuda.get_device_name(), "dtype": a.dtype, "num_q_heads": a.hq, "num_kv_heads": a.hkv,
           "head_dim": 128, "batch": BATCH, "kv_tokens": KV_TOTAL, "us": us, "heldout": held,
           "heldout_rel_err": {"median": statistics.median(errs), "max": max(errs)},
           "seconds": time.time() - t0}
    A.apex_cost_destroy(h)
    with open(a.out, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(doc["heldout_rel_err"]))


if __name__ == "__main__":
    main()
