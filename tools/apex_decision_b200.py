"""Feed APEX's decision layer (apex_decide: Eq5/Eq6 + Algorithm 1) with B200 numbers.

    python tools/apex_decision_b200.py [--batch 128 --ctx 8192] [--out profiles/apex_decision_b200.json]

* T_gatt   -- apex_predict_time on the calibrated table (profiles/cost_table_b200.json),
              per layer, for the batch's total KV tokens;
* T_glinear -- measured here: one LLaMA-3.1-8B layer's linear ops for `batch`
              decode tokens (QKV 4096x6144, O 4096x4096, gate+up 4096x28672,
              down 14336x4096; torch.matmul bf16 = cuBLAS, a plain library GEMM,
              not part of the hot path);
* N_G      -- kv_tokens / T_gatt;
* N_C      -- two CPU rates on this box's host: (a) the float64 oracle's measured
              rate (a floor: deliberately slow), (b) a bandwidth bound: host DRAM
              read bandwidth (numpy) / KV bytes per token (what an ideal
              memory-bound CPU kernel like the paper's Llamafile one could reach).
Prints and writes the Eq6 threshold, N_G/N_C and the decision for both N_C.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def t_glinear_us(batch, reps=50):
    import torch
    H, QKV, F = 4096, 6144, 14336
    x = torch.randn(batch, H, dtype=torch.bfloat16, device="cuda")
    w = {"qkv": torch.randn(H, QKV, dtype=torch.bfloat16, device="cuda"),
         "o": torch.randn(H, H, dtype=torch.bfloat16, device="cuda"),
         "gu": torch.randn(H, 2 * F, dtype=torch.bfloat16, device="cuda"),
         "d": torch.randn(F, H, dtype=torch.bfloat16, device="cuda")}
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def layer():
        y = x @ w["qkv"]
        z = x @ w["o"]
        g = x @ w["gu"]
        return (g[:, :F] @ w["d"]).sum() + y.sum() + z.sum()

    for _ in range(5):
        layer()
    ts = []
    for _ in range(reps):
        flush.zero_()                                  # weights come from HBM, as across layers
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        layer()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def host_read_gbs():
    import numpy as np
    a = np.ones(1 << 28, dtype=np.float64)      # 2 GiB
    a.sum()
    t = time.perf_counter()
    for _ in range(3):
        a.sum()
    return 3 * a.nbytes / (time.perf_counter() - t) / 1e9


def oracle_rate(ctx, hq, hkv):
    import synth
    from oracle import attention as oa
    q = synth.gen_rows(0, 0, [0], [ctx - 1], hq, 128, "bf16")
    k = synth.gen_seq(1, 0, 0, ctx, hkv, 128, "bf16")
    t = time.perf_counter()
    oa.decode_attention(q, [k], [k], "bf16", nthreads=len(os.sched_getaffinity(0)))
    return ctx / (time.perf_counter() - t) / 1e6          # tokens/us for one request, all heads


def main():
    from paper_2506_03296_b200 import apex as A
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--ctx", type=int, default=8192)
    ap.add_argument("--table", default=os.path.join(ROOT, "profiles", "cost_table_b200.json"))
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "apex_decision_b200.json"))
    a = ap.parse_args()
    tab = json.load(open(a.table))
    cost = A.apex_cost_create(tab["batch"], tab["kv_tokens"], tab["us"])
    kv = a.batch * a.ctx
    t_gatt = A.apex_predict_time(cost, a.batch, kv)
    t_lin = t_glinear_us(a.batch)
    n_g = kv / t_gatt
    kv_bytes_per_token = 2 * 8 * 128 * 2                      # K+V, 8 kv heads, bf16, one layer
    n_c_bw = host_read_gbs() * 1e9 / kv_bytes_per_token / 1e6 # tokens/us, bandwidth bound
    n_c_or = oracle_rate(a.ctx, 32, 8)
    res = {"batch": a.batch, "ctx": a.ctx, "kv_tokens": kv, "t_gatt_us": t_gatt, "t_glinear_us": t_lin,
           "n_g_tokens_per_us": n_g, "eq6_threshold": A.apex_pipelining_threshold(t_lin, t_gatt)}
    for name, n_c in (("cpu_bandwidth_bound", n_c_bw), ("cpu_oracle", n_c_or)):
        d = A.apex_decide(0, 0, a.batch * 8, n_g, n_c, t_lin, t_gatt, min_cpu_ratio=0.0)
        res[name] = {"n_c_tokens_per_us": n_c, "ng_over_nc": n_g / n_c, "decision": d["strategy"],
                     "eq5_lhs": d["lhs"], "eq5_rhs": d["rhs"]}
    A.apex_cost_destroy(cost)
    res["paper_reference"] = {"ng_over_nc_fig2b": 3031 / 170, "threshold_range": "5.83-7.5 for T_gatt/T_glinear in [0.5, 1.5] (P:203)"}
    print(json.dumps(res, indent=1))
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
