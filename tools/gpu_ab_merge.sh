#!/bin/bash
# Latency regime: decode kernel + a wide merge launch (ab/wide.so, -DAPEX_LAT_WIDE=1) vs the fused
# last-arriver merge (ab/pf.so): decode tests on the wide build, then same-box latency A/B.
set -u
O=gpurun_out/ab_merge6; mkdir -p $O
APEX_LIB=ab/wide.so timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_fused_append_gpu.py tests/test_graph_gpu.py tests/test_fused_gather_gpu.py -q -x > $O/tests.log 2>&1; echo "tests rc=$?"
for r in 1 2 3; do for v in pf wide; do
  APEX_LIB=ab/$v.so timeout 300 python tools/latency_probe.py --reps 25 > $O/lat_${v}_r$r.jsonl 2>&1
done; done
echo done
