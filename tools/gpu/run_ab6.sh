set -u
O=gpurun_out/ab6; mkdir -p $O
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_graph_gpu.py tests/test_configs_gpu.py -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?"
for c in c3 c5 c2 c4; do
for r in 1 2; do for lib in v1 swq32 swq48 swq20; do
APEX_LIB=ab/$lib.so timeout 600 python tools/tune.py --config $c --chunks 0 --reps 10 --scheds=-2,-1,-2:16/900/950/980,-2:32/900/950/980 | grep '^{"grid' | sed "s/^/$lib /" >> $O/tune_$c.log
done; done; done
