#!/bin/bash
# Same-box A/B of an environment variable read by bench.py or its dependencies (the library itself reads none), interleaved,
# under gpurun:  bash tools/ab_env.sh "<configs>" VAR "<values>"   -> gpurun_out/ab_env/
set -u
O=$PWD/gpurun_out/ab_env; mkdir -p $O
cfgs=$1; var=$2; vals=$3
for c in $cfgs; do for r in 1 2; do for v in $vals; do
  env $var=$v timeout 600 python bench.py --config $c --no-cpu --no-e2e --steps 10 > $O/${var}_${v}_${c}_$(date +%s%N).json 2>/dev/null
done; done; done
