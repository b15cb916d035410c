#!/bin/bash
# Guided-split chunk divisor sweep (apex_kv_set_planner guided_div; default 8 = T/(8P) tiles per
# piece, halved for the pairs holding the last 10/5/2% of the tiles): fewer, larger pieces mean
# fewer split pairs for the merge kernel and less per-item overhead, at the risk of imbalance.
set -u
O=gpurun_out/guided_div; mkdir -p $O
S="-2:8/900/950/980,-2:4/900/950/980,-2:2/900/950/980,-2:2/800/900/950,-2:1/900/950/980,-2:2/950/975/990"
for r in 1 2; do
  for c in c3 c2 c4 c5; do
    timeout 900 python tools/tune.py --config $c --chunks 0 --reps 20 --scheds=$S > $O/${c}_r$r.jsonl 2>&1
  done
done
echo done
