#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -m paper_2506_03296_b200.build > /dev/null
timeout 300 python tools/debug_signal2.py > gpurun_out/debug_signal2.txt 2>&1
O=gpurun_out/latency_variants.txt
for s in f32,32,32,1,512 bf16,32,8,1,16384 bf16,32,8,64,1024 bf16,32,8,16,2048 bf16,32,8,256,512; do
  python tools/latency_probe.py --shape $s >> $O 2>&1
  python tools/latency_probe.py --shape $s --graph >> $O 2>&1
  python tools/latency_probe.py --shape $s --lat-tiles 0 >> $O 2>&1
  python tools/latency_probe.py --shape $s --lat-tiles 0 --sched 0 >> $O 2>&1
  python tools/latency_probe.py --shape $s --lat-tiles 0 --sched 100 >> $O 2>&1
done
