"""Copy/summarise gpurun_out/refresh/ (tools/refresh_profiles.sh) into profiles/ (round tag).

    python tools/ingest_refresh.py [--src gpurun_out/refresh] [--tag r02]

Prints the results table used in DESIGN.md §8.
"""
import argparse
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--src", default=os.path.join(ROOT, "gpurun_out", "refresh"))
    ap.add_argument("--tag", default="r02")
    a = ap.parse_args()
    prof = os.path.join(ROOT, "profiles")
    src = a.src
    cp = lambda f, d: os.path.exists(os.path.join(src, f)) and shutil.copy(os.path.join(src, f), os.path.join(prof, d))
    for c in ("c1", "c2", "c3", "c4", "c5"):
        cp(f"bench_{c}.json", f"{a.tag}_{c}_bench.json")
        rep = os.path.join(src, f"prof_{c}.ncu-rep")
        if os.path.exists(rep):
            # key = bench.py's (config, mode, N) lookup for roofline.traffic (N = 1: request mode)
            subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), "--tag", f"{a.tag}_{c}",
                            "--config", f"{c}:req:1", "--rep", rep], check=True, capture_output=True)
            shutil.copy(rep, os.path.join(prof, f"{a.tag}_{c}_decode.ncu-rep"))
    cp("bench_reference_c5.json", f"{a.tag}_c5_reference_bench.json")
    cp("bench_c5_eager.json", f"{a.tag}_c5_eager_bench.json")
    cp("bench_c5_head1.json", f"{a.tag}_c5_head1_nccl_bench.json")
    cp("latency_probe.jsonl", f"{a.tag}_latency_probe_final.jsonl")
    cp("gpus2_head.json", f"{a.tag}_gpus2_head_same_gpu.json")
    cp("gpus2_req.json", f"{a.tag}_gpus2_req_same_gpu.json")
    cp("clocks_before.txt", f"{a.tag}_refresh_clocks_before.txt")
    for name, tag in (("launches_c5_timed.csv", "c5_timed"),):
        f = os.path.join(src, name)
        if os.path.exists(f):
            subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), "--tag", f"{a.tag}_{tag}",
                            "--config", tag, "--launches", f], check=True, capture_output=True)
    cp("hbm_probe.txt", f"{a.tag}_hbm_read_probe.txt")
    cp("pytest_gpu.log", f"{a.tag}_pytest_gpu_full.log")
    cp("smoke.log", f"{a.tag}_smoke.log")
    rows = []
    for c in ("c1", "c2", "c3", "c4", "c5"):
        f = os.path.join(prof, f"{a.tag}_{c}_bench.json")
        if not os.path.exists(f):
            continue
        d = json.load(open(f))
        r, p, cb = d["roofline"], d.get("parity_sample", {}), d.get("cpu_baseline", {})
        rows.append(f"| {c.upper()} | {d['details']['phys_layers']} | {d['value']:.0f} | {d['ms_per_step']:.3f} | "
                    f"{r['avg_launch_us']:.1f} | {r['achieved']:.0f} | {r['frac']:.3f} | {r['frac_of_8000_gbs']:.3f} | "
                    f"{d['e2e']['value']:.0f} | {cb.get('value', 0):.3g} ({cb.get('cores', '?')} thr) | "
                    f"{p.get('max_abs_err', 0):.1e} | {d.get('clocks', {}).get('sm_mhz', '?')} |")
    print("\n".join(rows))


if __name__ == "__main__":
    main()
