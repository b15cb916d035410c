#!/bin/bash
# Partial refresh under gpurun: bench.py for the given configs (+ smoke) into gpurun_out/refresh/.
#   bash tools/refresh_partial.sh "c1 c3"
set -u
O=gpurun_out/refresh; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
for c in $1; do
  timeout 600 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?"
done
