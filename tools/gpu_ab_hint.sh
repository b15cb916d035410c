#!/bin/bash
# Same-box A/B of the mbarrier try_wait suspend-time hint (ab/hint<ns>.so) vs none (ab/cur.so):
# sustained benches (power-capped) and latency-regime calls.
set -u
O=gpurun_out/ab_hint; mkdir -p $O
for r in 1 2; do for v in cur hint1000 hint20000 hint1000000; do
  APEX_LIB=ab/$v.so timeout 600 python bench.py --no-cpu --no-e2e > $O/c5_${v}_r$r.json 2>/dev/null
  APEX_LIB=ab/$v.so timeout 600 python bench.py --config c3 --steps 60 --no-cpu --no-e2e > $O/c3_${v}_r$r.json 2>/dev/null
done; done
for v in cur hint20000 hint1000000; do
  APEX_LIB=ab/$v.so timeout 300 python tools/latency_probe.py --reps 25 > $O/lat_${v}.jsonl 2>&1
done
echo done
