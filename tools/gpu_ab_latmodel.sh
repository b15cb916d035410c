#!/bin/bash
# Latency-regime chunk model: current (ab/lat0.so) vs concurrency-aware (ab/lat1.so, -DAPEX_LAT_MODEL=1),
# tools/latency_probe.py (L2 read-flushed), interleaved, two rounds.
set -u
O=gpurun_out/ab_latmodel; mkdir -p $O
for r in 1 2; do for v in lat0 lat1; do
  APEX_LIB=ab/$v.so timeout 600 python tools/latency_probe.py --reps 25 > $O/${v}_r$r.jsonl 2>&1
done; done
echo done
