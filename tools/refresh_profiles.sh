#!/bin/bash
# Regenerate the measured artifacts of profiles/ on a GPU box (run under gpurun):
# GPU test suite + smoke, bench.py c5 (default line) + reference arm, c1..c4 lines,
# ncu --set full of the decode kernel per config, the timed-step launch list of the
# default bench, the latency probe, the 2-rank same-GPU logic runs and the HBM read
# probe.  Outputs land in gpurun_out/refresh/; tools/ingest_refresh.py copies them.
set -u
O=gpurun_out/refresh
mkdir -p $O
nvidia-smi -q -d CLOCK > $O/clocks_before.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; echo "bench c5 rc=$?"
timeout 600 python bench.py --impl reference > $O/bench_reference_c5.json 2> $O/bench_reference_c5.err; echo "ref rc=$?"
timeout 900 python bench.py --launch eager --no-cpu > $O/bench_c5_eager.json 2> $O/bench_c5_eager.err; echo "bench c5 eager rc=$?"
timeout 900 python bench.py --mode head --no-cpu > $O/bench_c5_head1.json 2> $O/bench_c5_head1.err; echo "bench c5 head1 rc=$?"
for c in c3 c1 c2 c4; do
  timeout 600 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?"
done
timeout 600 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_c5_timed.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1; echo "launches rc=$?"
for c in c5 c3 c2 c4; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:apex_decode_kernel -s 40 -c 1 \
    -o $O/prof_$c python bench.py --config $c --steps 2 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1; echo "ncu $c rc=$?"
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:apex_decode_kernel -s 2 -c 1 \
  -o $O/prof_c1 python bench.py --config c1 --steps 2 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1; echo "ncu c1 rc=$?"
timeout 600 python tools/latency_probe.py --reps 25 > $O/latency_probe.jsonl 2>&1; echo "latency rc=$?"
timeout 900 python bench.py --gpus 2 --steps 5 > $O/gpus2_head.json 2> $O/gpus2_head.err; echo "gpus2 head rc=$?"
timeout 900 python bench.py --gpus 2 --steps 5 --mode req > $O/gpus2_req.json 2> $O/gpus2_req.err; echo "gpus2 req rc=$?"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/hbm_probe.cu -o /tmp/hbm_probe 2>/dev/null && \
  timeout 120 /tmp/hbm_probe > $O/hbm_probe.txt 2>&1; echo "probe rc=$?"
nvidia-smi -q -d CLOCK > $O/clocks_after.txt 2>&1
