"""Where does the end-to-end (host buffers) time go?  One C3 layer, repeated.

    python tools/e2e_probe.py [--layers 32]

Times L layer-calls of (append + decode) with inputs resident (device), with
pinned-host inputs/outputs copied on the compute stream (serial), and with the
copies on a second stream double-buffered underneath the previous layer
(overlapped, what bench.py's e2e leg does).  Also reports the host enqueue time.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch

    from helpers import gen_dev, make_cache, prefill
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--ctx", type=int, default=8192)
    a = ap.parse_args()
    B, L = a.batch, a.layers
    cache = make_cache("bf16", 32, 8, B * (a.ctx // 16 + 8), max_seqs=B, max_blocks_per_seq=a.ctx // 16 + 8)
    seqs = list(range(B))
    prefill(cache, seqs, [a.ctx] * B)
    pos = [a.ctx - 1] * B
    q = gen_dev(cache, 0, 0, seqs, pos, 32)
    k = gen_dev(cache, 1, 0, seqs, pos, 8)
    v = gen_dev(cache, 2, 0, seqs, pos, 8)
    out = torch.empty_like(q)
    qh, kh, vh = (t.cpu().pin_memory() for t in (q, k, v))
    oh = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
    qd = [torch.empty_like(q) for _ in range(2)]
    kd = [torch.empty_like(k) for _ in range(2)]
    vd = [torch.empty_like(v) for _ in range(2)]
    od = [torch.empty_like(out) for _ in range(2)]
    comp, copy, d2h_s = torch.cuda.current_stream(), torch.cuda.Stream(), torch.cuda.Stream()
    h2d = [torch.cuda.Event() for _ in range(2)]
    dec = [torch.cuda.Event() for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]
    for e in free:
        e.record(comp)

    def resident():
        cache.alloc(seqs, [1] * B)
        for _ in range(L):
            cache.append(0, k, v)
            cache.decode(0, q, out=out)

    def serial():
        cache.alloc(seqs, [1] * B)
        for _ in range(L):
            qd[0].copy_(qh, non_blocking=True)
            kd[0].copy_(kh, non_blocking=True)
            vd[0].copy_(vh, non_blocking=True)
            cache.append(0, kd[0], vd[0])
            cache.decode(0, qd[0], out=od[0])
            oh.copy_(od[0], non_blocking=True)

    def overlapped():
        cache.alloc(seqs, [1] * B)
        for l in range(L):
            j = l % 2
            with torch.cuda.stream(copy):
                copy.wait_event(free[j])
                qd[j].copy_(qh, non_blocking=True)
                kd[j].copy_(kh, non_blocking=True)
                vd[j].copy_(vh, non_blocking=True)
                h2d[j].record(copy)
            comp.wait_event(h2d[j])
            cache.append(0, kd[j], vd[j])
            cache.decode(0, qd[j], out=od[j])
            dec[j].record(comp)
            with torch.cuda.stream(d2h_s):
                d2h_s.wait_event(dec[j])
                oh.copy_(od[j], non_blocking=True)
                free[j].record(d2h_s)
        for e in free:
            comp.wait_event(e)

    def copies_only():
        for _ in range(L):
            qd[0].copy_(qh, non_blocking=True)
            kd[0].copy_(kh, non_blocking=True)
            vd[0].copy_(vh, non_blocking=True)
            oh.copy_(od[0], non_blocking=True)

    res = {}
    for name, fn in (("resident", resident), ("serial", serial), ("overlapped", overlapped),
                     ("copies_only", copies_only)):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        for _ in range(5):
            fn()
        t_host = (time.perf_counter() - t0) / 5
        e1.record()
        torch.cuda.synchronize()
        res[name] = {"gpu_ms_per_step": e0.elapsed_time(e1) / 5, "host_enqueue_ms_per_step": t_host * 1e3}
        print(name, res[name], flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
