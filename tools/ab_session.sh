#!/bin/bash
# Same-box A/B under gpurun: git worktrees of earlier commits (ab/old_tree = session start)
# against the current tree, bench.py lines interleaved.  Output: gpurun_out/ab_session5/
set -u
O=$PWD/gpurun_out/ab_session5; mkdir -p $O
run() { local tag=$1; shift; timeout 600 "$@" > $O/${tag}_$(date +%s%N).json 2>/dev/null; }
for c in c5 c2 c3; do
  for r in 1 2; do
    (cd ab/old_tree && run old_$c python bench.py --config $c --no-cpu --no-e2e --steps 10)
    run cursep_$c python bench.py --config $c --no-cpu --no-e2e --steps 10 --append separate
    run curfused_$c python bench.py --config $c --no-cpu --no-e2e --steps 10
  done
done
