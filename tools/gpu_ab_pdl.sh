#!/bin/bash
# Upload kernel triggering programmatic dependents at its start (ab/pdl.so = in-tree) vs not
# (ab/nopdl.so): GPU suite subset on the in-tree build, then C1 / alloc_probe, interleaved.
set -u
O=gpurun_out/ab_pdl; mkdir -p $O
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_graph_gpu.py tests/test_fused_append_gpu.py tests/test_bounds_gpu.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"
for r in 1 2; do for v in nopdl pdl; do
  APEX_LIB=ab/$v.so timeout 300 python tools/alloc_probe.py > $O/alloc_${v}_r$r.jsonl 2>&1
  for m in graph eager; do
    APEX_LIB=ab/$v.so timeout 300 python bench.py --config c1 --launch $m --no-cpu --no-e2e > $O/c1_${v}_${m}_r$r.json 2>/dev/null
  done
done; done
echo done
