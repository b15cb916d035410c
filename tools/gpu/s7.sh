#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/s7; mkdir -p $O
python -m paper_2506_03296_b200.build > /dev/null
timeout 300 python -m pytest tests/test_decode_gpu.py -q -k "two_level" > $O/pytest_two_level.log 2>&1; echo "two_level rc=$?" >> $O/rc.txt
python tools/latency_probe.py > $O/latency_probe.txt 2>&1
python -m paper_2506_03296_b200.build -DAPEX_TRACE --out=/tmp/trace.so > /dev/null 2>&1
for s in bf16,32,8,1,16384 f32,32,32,1,512; do
  APEX_LIB=/tmp/trace.so python tools/trace_probe.py --shape $s >> $O/trace.txt 2>&1
done
timeout 900 python bench.py --gpus 2 --steps 5 > $O/bench_gpus2_head.json 2> $O/bench_gpus2_head.err; echo "g2h rc=$?" >> $O/rc.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
