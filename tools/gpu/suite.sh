#!/bin/bash
# GPU-box session: build, smoke, GPU tests, default bench (C5 N=1), 2-rank same-device
# logic runs of the sharded paths.  Outputs land in gpurun_out/ (merged back by gpurun).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
if [ -z "$SKIP_BENCH" ]; then
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
fi
if [ -n "$MULTI" ]; then
timeout 900 python bench.py --gpus 2 --steps 5 > gpurun_out/bench_gpus2_head.json 2> gpurun_out/bench_gpus2_head.err; echo "rc=$?" >> gpurun_out/bench_gpus2_head.err
timeout 900 python bench.py --gpus 2 --steps 5 --mode req > gpurun_out/bench_gpus2_req.json 2> gpurun_out/bench_gpus2_req.err; echo "rc=$?" >> gpurun_out/bench_gpus2_req.err
fi
