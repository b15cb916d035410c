"""f4: the Asynchronous-Overlap idea (§3.3) mapped onto one B200.

APEX overlaps CPU attention of one set of requests with GPU linear layers of the
whole batch, because the CPU's DRAM bandwidth is *additional* to the GPU's.  On a
single B200 the analogue is intra-device overlap: decode attention for half of
the batch (apex_decode_attention, HBM-bound) on one stream while the other half's
linear layers (cuBLAS bf16 GEMMs of one LLaMA-3.1-8B layer) run on another.

    python tools/overlap_b200.py [--batch 128 --ctx 8192] [--att-grid 148]

Reports serial vs concurrent time for one layer's worth of work and the
overlap gain.  The attention grid can be capped (apex_kv_set_grid) so GEMM CTAs
find free SM resources.  Output: profiles/apex_overlap_b200.json.
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
    import torch

    from helpers import gen_dev, make_cache, prefill
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--ctx", type=int, default=8192)
    ap.add_argument("--att-grid", type=int, default=0, help="persistent CTAs for attention (0 = default 2/SM)")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "apex_overlap_b200.json"))
    a = ap.parse_args()
    half = a.batch // 2
    cache = make_cache("bf16", 32, 8, half * (a.ctx // 16 + 2), max_seqs=half, max_blocks_per_seq=a.ctx // 16 + 2)
    seqs = list(range(half))
    prefill(cache, seqs, [a.ctx] * half)
    cache.alloc(seqs, [1] * half)
    k = gen_dev(cache, 1, 0, seqs, [a.ctx - 1] * half, 8)
    cache.append(0, k, k)
    q = gen_dev(cache, 0, 0, seqs, [a.ctx - 1] * half, 32)
    out = torch.empty_like(q)
    H, QKV, F = 4096, 6144, 14336
    x = torch.randn(half, H, dtype=torch.bfloat16, device="cuda")
    w = [torch.randn(H, QKV, dtype=torch.bfloat16, device="cuda"), torch.randn(H, H, dtype=torch.bfloat16, device="cuda"),
         torch.randn(H, 2 * F, dtype=torch.bfloat16, device="cuda"), torch.randn(F, H, dtype=torch.bfloat16, device="cuda")]
    g_in = torch.randn(half, F, dtype=torch.bfloat16, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def linear():
        x @ w[0]
        x @ w[1]
        x @ w[2]
        g_in @ w[3]

    def attention():
        cache.decode(0, q, out=out)

    s_att, s_lin = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        ts = []
        for r in range(a.reps + 3):
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if r >= 3:
                ts.append(e0.elapsed_time(e1) * 1e3)
        return statistics.median(ts)

    def concurrent():
        cur = torch.cuda.current_stream()
        s_att.wait_stream(cur)
        s_lin.wait_stream(cur)
        with torch.cuda.stream(s_att):
            attention()
        with torch.cuda.stream(s_lin):
            linear()
        cur.wait_stream(s_att)
        cur.wait_stream(s_lin)

    res = {"batch_half": half, "ctx": a.ctx}
    for grid in sorted({0, a.att_grid, 148}):
        cache.set_grid(grid)
        cache.alloc(seqs, [0] * half)              # re-plan for this grid
        t_att = timed(attention)
        t_lin = timed(linear)
        t_ser = timed(lambda: (attention(), linear()))
        t_con = timed(concurrent)
        res[f"grid_{grid or 'default'}"] = {"attention_us": t_att, "linear_us": t_lin, "serial_us": t_ser,
                                            "concurrent_us": t_con, "gain": t_ser / t_con - 1.0,
                                            "ideal_gain": t_ser / max(t_att, t_lin) - 1.0}
    print(json.dumps(res, indent=1))
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
