#!/bin/bash
# Full GPU session: build, smoke, pytest -m gpu, default bench (C5 N=1), reference arm,
# 2-rank same-GPU sharded runs, calibrated cost table.  Outputs in gpurun_out/round/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/round; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?" >> $O/rc.txt
timeout 900 python bench.py --gpus 2 --steps 5 > $O/bench_gpus2_head.json 2> $O/bench_gpus2_head.err; echo "g2h rc=$?" >> $O/rc.txt
timeout 900 python bench.py --gpus 2 --steps 5 --mode req > $O/bench_gpus2_req.json 2> $O/bench_gpus2_req.err; echo "g2r rc=$?" >> $O/rc.txt
if [ -n "$CALIB" ]; then
timeout 1500 python tools/calibrate.py --out $O/cost_table_b200.json > $O/calibrate.log 2>&1; echo "calib rc=$?" >> $O/rc.txt
fi
