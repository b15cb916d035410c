"""Summarise ncu outputs brought back in gpurun_out/ into profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py --tag r01_c3 --config c3 --launches gpurun_out/launches_c3.csv \
        --rep gpurun_out/prof_c3.ncu-rep [--bench gpurun_out/bench_c3.json]

Writes profiles/<tag>_launches.txt (per-kernel count / total / avg / share of the
launch list), profiles/<tag>_ncu_full.txt (key --set full metrics of the captured
decode launch) and updates profiles/ncu_summary.json[config] with the decode
kernel's DRAM bytes per launch (bench.py's roofline.traffic).
"""
import argparse
import collections
import csv
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes.sum.per_second",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second", "dram__cycles_elapsed.avg.per_second",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    agg = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}[d["Metric Unit"]]
        name = d["Kernel Name"].split("(")[0]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    lines = [f"{'kernel':70s} {'n':>6s} {'total_ms':>10s} {'avg_us':>10s} {'share':>6s}"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{k[:70]:70s} {n:6d} {t / 1e3:10.3f} {t / n:10.2f} {t / tot:6.3f}")
    return "\n".join(lines)


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    res = []
    for v in vals:
        d = {}
        for i, k in enumerate(hdr):
            if k in KEYS or k in ("Kernel Name",):
                d[k] = (v[i], units[i])
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--config", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--bench")
    a = ap.parse_args()
    prof = os.path.join(ROOT, "profiles")
    if a.launches:
        txt = launches(a.launches)
        open(os.path.join(prof, f"{a.tag}_launches.txt"), "w").write(
            f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised; compare shares)\n"
            f"# source: {os.path.basename(a.launches)}\n" + txt + "\n")
        print(txt)
    if a.rep:
        caps = full(a.rep)
        lines = []
        for d in caps:
            for k in ["Kernel Name"] + KEYS:
                if k in d:
                    lines.append(f"{k:62s} {d[k][1]:>12s} {d[k][0]}")
            lines.append("")
        open(os.path.join(prof, f"{a.tag}_ncu_full.txt"), "w").write(
            "# ncu --set full --clock-control none --import-source on -k regex:apex_decode_kernel (one launch)\n"
            + "\n".join(lines))
        print("\n".join(lines))
        d = caps[0]
        rd = float(d["dram__bytes_read.sum"][0]) * SCALE[d["dram__bytes_read.sum"][1]]
        wr = float(d["dram__bytes_write.sum"][0]) * SCALE[d["dram__bytes_write.sum"][1]]
        sp = os.path.join(prof, "ncu_summary.json")
        summ = json.load(open(sp)) if os.path.exists(sp) else {}
        summ[a.config] = {"decode_dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                          "duration_us": float(d["gpu__time_duration.sum"][0]) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[d["gpu__time_duration.sum"][1]], "tag": a.tag}
        json.dump(summ, open(sp, "w"), indent=1)
    if a.bench:
        import shutil
        shutil.copy(a.bench, os.path.join(prof, f"{a.tag}_bench.json"))


if __name__ == "__main__":
    main()
