#!/bin/bash
# Same-box A/B of libapex builds (APEX_LIB=ab/<name>.so) with bench.py, interleaved, under gpurun.
#   bash tools/ab_libs.sh "<configs>" <lib1> <lib2> ...   -> gpurun_out/ab_libs/
set -u
O=$PWD/gpurun_out/ab_libs; mkdir -p $O
cfgs=$1; shift
for c in $cfgs; do for r in 1 2; do for v in "$@"; do
  APEX_LIB=ab/$v.so timeout 600 python bench.py --config $c --no-cpu --steps 10 > $O/${v}_${c}_$(date +%s%N).json 2>/dev/null
done; done; done
