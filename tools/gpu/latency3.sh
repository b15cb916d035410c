#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -m paper_2506_03296_b200.build > /dev/null
python tools/launch_floor.py > gpurun_out/launch_floor.txt 2>&1
for f in read write; do python tools/latency_probe.py --flush $f > gpurun_out/latency_probe_$f.txt 2>&1; done
