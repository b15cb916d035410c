#!/bin/bash
# Regenerate every measured artifact of profiles/ on a GPU box (run under gpurun):
# benches for c1..c5, ncu --set full of the decode kernel per config, the timed-step
# launch list of the default bench, the calibrated cost table, the APEX decision,
# the HBM read probe and the GPU test log.  Outputs land in gpurun_out/refresh/.
set -u
O=gpurun_out/refresh
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
for c in c3 c1 c2 c4 c5; do
  timeout 600 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?"
done
timeout 300 python bench.py --impl reference > $O/bench_reference_c3.json 2> $O/bench_reference_c3.err; echo "ref rc=$?"
for c in c2 c3 c4 c5; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:apex_decode_kernel -s 40 -c 1 \
    -o $O/prof_$c python bench.py --config $c --steps 2 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1; echo "ncu $c rc=$?"
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:apex_decode_kernel -s 2 -c 1 \
  -o $O/prof_c1 python bench.py --config c1 --steps 2 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1; echo "ncu c1 rc=$?"
timeout 300 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_c3_timed.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1; echo "launches rc=$?"
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $O/launches_c3_all.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1; echo "launches-all rc=$?"
timeout 900 python tools/calibrate.py --out $O/cost_table_b200.json > $O/calibrate.log 2>&1; echo "calibrate rc=$?"
timeout 300 python tools/apex_decision_b200.py --table $O/cost_table_b200.json --out $O/apex_decision_b200.json > $O/decision.log 2>&1; echo "decision rc=$?"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/hbm_probe.cu -o /tmp/hbm_probe 2>/dev/null && timeout 120 /tmp/hbm_probe > $O/hbm_probe.txt 2>&1; echo "probe rc=$?"
