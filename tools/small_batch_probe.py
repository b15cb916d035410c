"""Decode-call latency for few, long sequences (the merge fan-in regime).

    python tools/small_batch_probe.py
Prints us per apex_decode_attention (L2 flushed) for batch x per-request context.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    import torch

    from calibrate import measure
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    res = []
    for b, ctx in [(1, 16384), (1, 65536), (1, 262144), (4, 16384), (4, 65536), (16, 16384), (64, 4096)]:
        us, kv = measure("bf16", 32, 8, b, b * ctx, 7, flush)
        gbs = kv * 8 * 128 * 2 * 2 / us / 1e3
        res.append({"batch": b, "ctx": ctx, "us": us, "gbs": gbs})
        print(json.dumps(res[-1]), flush=True)


if __name__ == "__main__":
    main()
