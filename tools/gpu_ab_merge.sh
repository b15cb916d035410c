#!/bin/bash
# Warp-per-row LSE merge (ab/v2.so, in-tree build) vs the running-max fold (ab/pf.so):
# GPU decode tests on the in-tree build, then same-box latency / bandwidth A/B and traces.
set -u
O=gpurun_out/ab_merge3; mkdir -p $O
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_fused_append_gpu.py tests/test_graph_gpu.py tests/test_fused_gather_gpu.py tests/test_wide_range_gpu.py -q -x > $O/tests.log 2>&1; echo "tests rc=$?"
for r in 1 2; do for v in pf v2; do
  APEX_LIB=ab/$v.so timeout 300 python tools/latency_probe.py --reps 25 > $O/lat_${v}_r$r.jsonl 2>&1
done; done
for v in pftr v2tr; do for s in bf16,32,8,1,16384 f32,32,32,1,512 bf16,32,8,1,4096; do
  APEX_LIB=ab/$v.so timeout 120 python tools/trace_probe.py --shape $s >> $O/trace_$v.jsonl 2>&1
done; done
for c in c3 c2; do for r in 1 2; do for v in pf v2; do
  APEX_LIB=ab/$v.so timeout 300 python tools/tune.py --config $c --chunks 0 --reps 20 2>&1 | grep '"grid"' > $O/tune_${c}_${v}_r$r.txt
done; done; done
echo done
