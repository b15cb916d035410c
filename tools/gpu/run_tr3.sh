set -u
O=gpurun_out/tr3; mkdir -p $O; rm -f $O/trace.log
for lib in trace trace_u4; do for sh in f32,32,32,1,512 bf16,32,8,1,16384; do
APEX_LIB=ab/$lib.so timeout 300 python tools/trace_probe.py --shape $sh | sed "s/^/$lib flush /" >> $O/trace.log 2>&1
APEX_LIB=ab/$lib.so timeout 300 python tools/trace_probe.py --shape $sh --no-flush | sed "s/^/$lib warm /" >> $O/trace.log 2>&1
done; done
for lib in m3 m4; do
APEX_LIB=ab/$lib.so timeout 600 python tools/latency_probe.py | sed "s/^/$lib /" >> $O/lat.log
done
timeout 900 python -m pytest tests/test_decode_gpu.py -q -m gpu -x > $O/pytest.log 2>&1; echo "pytest rc=$?"
