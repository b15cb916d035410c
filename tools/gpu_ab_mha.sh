#!/bin/bash
# Sustained (power-capped) A/B of the bandwidth-regime 16-bit MHA consumer: CUDA cores (ab/cur.so)
# vs the transposed tensor-core path with one live head column (ab/mhatc.so, -DAPEX_MHA_TC_BW=1).
set -u
O=gpurun_out/ab_mha; mkdir -p $O
for r in 1 2 3; do for v in cur mhatc; do
  APEX_LIB=ab/$v.so timeout 600 python bench.py --config c2 --steps 60 --no-cpu --no-e2e > $O/bench_${v}_r$r.json 2>/dev/null
done; done
for r in 1 2; do for v in cur mhatc; do
  APEX_LIB=ab/$v.so timeout 300 python tools/tune.py --config c2 --chunks 0 --reps 20 2>&1 | grep '"grid"' > $O/tune_${v}_r$r.txt
done; done
echo done
