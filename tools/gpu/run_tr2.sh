set -u
O=gpurun_out/tr2; mkdir -p $O
for sh in f32,32,32,1,512 bf16,32,8,1,16384; do
APEX_LIB=ab/trace.so timeout 300 python tools/trace_probe.py --shape $sh >> $O/trace.log 2>&1
done
