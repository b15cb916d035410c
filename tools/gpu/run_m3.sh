set -u
O=gpurun_out/m3; mkdir -p $O
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_graph_gpu.py -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?"
for lib in m2 m3 m2 m3; do
APEX_LIB=ab/$lib.so timeout 600 python tools/latency_probe.py | sed "s/^/$lib /" >> $O/lat.log
done
for lib in m2 m3; do
APEX_LIB=ab/$lib.so timeout 600 python tools/tune.py --config c3 --chunks 0 --reps 10 | grep '^{"grid' | sed "s/^/$lib /" >> $O/tune_c3.log
done
for sh in f32,32,32,1,512 bf16,32,8,1,16384; do
APEX_LIB=ab/trace.so timeout 300 python tools/trace_probe.py --shape $sh >> $O/trace.log 2>&1
done
