set -u
O=gpurun_out/cl1; mkdir -p $O
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_graph_gpu.py -q -m gpu -x > $O/pytest.log 2>&1; echo "pytest rc=$?"
for lib in m2 cl; do
APEX_LIB=ab/$lib.so timeout 600 python tools/latency_probe.py | sed "s/^/$lib /" >> $O/lat.log
done
for sh in f32,32,32,1,512 bf16,32,8,1,16384 bf16,32,8,4,4096; do
APEX_LIB=ab/trace.so timeout 300 python tools/trace_probe.py --shape $sh >> $O/trace.log 2>&1
done
