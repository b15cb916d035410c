set -u
O=gpurun_out/ab2; mkdir -p $O
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_graph_gpu.py -q -m gpu -x > $O/pytest.log 2>&1; echo "pytest rc=$?"
for c in c3 c2 c4 c5; do
for r in 1 2; do for lib in v1 v2 v2far; do
APEX_LIB=ab/$lib.so timeout 600 python tools/tune.py --config $c --chunks 0 --reps 15 --scheds=-2,-2:16/900/950/980,-1 | grep '^{"grid' | sed "s/^/$lib /" >> $O/tune_$c.log
done; done; done
