#!/bin/bash
# Host-side alloc speedups (scratch reuse, per-(length, chunk) pieces, counting sort, numpy
# marshalling) + single-launch zero-copy upload (ab/new.so = in-tree) vs the round's earlier
# library (ab/copy.so: per-step vectors, stable_sort, H2D copy + delta kernel): GPU suite on
# the in-tree build, then tools/alloc_probe.py and C1 benches, interleaved.
set -u
O=gpurun_out/ab_host; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"
for r in 1 2; do for v in copy new; do
  APEX_LIB=ab/$v.so timeout 300 python tools/alloc_probe.py > $O/alloc_${v}_r$r.jsonl 2>&1
  APEX_LIB=ab/$v.so timeout 300 python bench.py --config c1 --no-cpu > $O/c1_${v}_r$r.json 2>/dev/null
done; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
echo done
