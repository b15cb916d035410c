#!/bin/bash
# latency-regime session: launch floor, latency probe, per-CTA traces (APEX_TRACE build in /tmp)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -m paper_2506_03296_b200.build > /dev/null
python tools/launch_floor.py > gpurun_out/latency_floor.json 2>&1
python tools/latency_probe.py > gpurun_out/latency_probe.txt 2>&1
python -m paper_2506_03296_b200.build -DAPEX_TRACE --out=/tmp/trace.so > /dev/null 2>&1
for s in f32,32,32,1,512 bf16,32,8,1,16384 bf16,32,8,64,1024 bf16,32,8,1,512; do
  APEX_LIB=/tmp/trace.so python tools/trace_probe.py --shape $s >> gpurun_out/latency_trace.txt 2>&1
done
