#!/bin/bash
# Single-launch zero-copy metadata upload (ab/upk.so = in-tree) vs H2D copy + delta kernel
# (ab/copy.so, -DAPEX_UPLOAD_KERNEL=0): GPU suite on the in-tree build, then per-piece step
# times (tools/alloc_probe.py) and same-box benches, interleaved.
set -u
O=gpurun_out/ab_upload; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"
for r in 1 2; do for v in copy upk; do
  APEX_LIB=ab/$v.so timeout 300 python tools/alloc_probe.py > $O/alloc_${v}_r$r.jsonl 2>&1
  APEX_LIB=ab/$v.so timeout 300 python bench.py --config c1 --no-cpu > $O/c1_${v}_r$r.json 2>/dev/null
done; done
for v in copy upk; do
  APEX_LIB=ab/$v.so timeout 600 python bench.py --config c3 --no-cpu --no-e2e > $O/c3_${v}.json 2>/dev/null
  APEX_LIB=ab/$v.so timeout 900 python bench.py --no-cpu --no-e2e > $O/c5_${v}.json 2>/dev/null
done
echo done
