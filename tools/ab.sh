#!/bin/bash
# A/B decode timing of several libapex builds on the same GPU, interleaved:
#   tools/ab.sh <config> <chunks> lib1.so lib2.so ...
cfg=$1; chunks=$2; shift 2
for round in 1 2; do
  for lib in "$@"; do
    echo "== $lib round $round"
    APEX_LIB=$lib timeout 300 python tools/tune.py --config $cfg --chunks $chunks --reps 20 | grep -v '^{"config'
  done
done
