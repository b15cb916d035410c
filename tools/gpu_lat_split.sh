#!/bin/bash
# Latency regime: the planner's chunk (fused merge) vs forced chunks (whole pairs = no merge,
# one launch; split chunks = merge-kernel launch) on small shapes, L2 read-flushed.
set -u
O=gpurun_out/lat_split; mkdir -p $O
for shp in f32,32,32,1,512 bf16,32,8,1,512 f16,32,32,8,1024 bf16,32,8,64,1024 bf16,32,8,16,2048; do
  for sp in 0 64 128 256 512 1024 2048; do
    timeout 300 python tools/latency_probe.py --reps 25 --shape $shp --split $sp >> $O/split.jsonl 2>/dev/null
  done
done
for g in 148 296 444; do
  timeout 300 python tools/latency_probe.py --reps 25 --shape f32,32,32,1,512 --split 528 >> $O/grid.jsonl 2>/dev/null
done
echo done
