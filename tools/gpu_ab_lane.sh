#!/bin/bash
# Lane-parallel producer (ab/lane.so = in-tree; lane w < NC refills consumer warp w's sub-ring) vs one
# issuing lane (ab/cur.so): full GPU suite on the in-tree build, then sustained same-box benches.
set -u
O=gpurun_out/ab_lane; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"
for r in 1 2 3; do for v in cur lane; do
  APEX_LIB=ab/$v.so timeout 600 python bench.py --no-cpu --no-e2e > $O/c5_${v}_r$r.json 2>/dev/null
  APEX_LIB=ab/$v.so timeout 600 python bench.py --config c3 --steps 60 --no-cpu --no-e2e > $O/c3_${v}_r$r.json 2>/dev/null
done; done
for r in 1 2; do for v in cur lane; do
  APEX_LIB=ab/$v.so timeout 600 python bench.py --config c2 --steps 60 --no-cpu --no-e2e > $O/c2_${v}_r$r.json 2>/dev/null
  APEX_LIB=ab/$v.so timeout 600 python bench.py --config c4 --steps 10 --no-cpu --no-e2e > $O/c4_${v}_r$r.json 2>/dev/null
done; done
for v in cur lane; do
  APEX_LIB=ab/$v.so timeout 300 python tools/latency_probe.py --reps 25 > $O/lat_${v}.jsonl 2>&1
done
echo done
