set -u
O=gpurun_out/lat1; mkdir -p $O
for r in 1 2; do for lib in v1 swq32; do
APEX_LIB=ab/$lib.so timeout 600 python tools/latency_probe.py | sed "s/^/$lib /" >> $O/lat.log
done; done
timeout 600 python bench.py --config c1 > $O/bench_c1.json 2> $O/bench_c1.err
APEX_LIB=ab/v1.so timeout 600 python bench.py --config c1 > $O/bench_c1_v1.json 2> $O/bench_c1_v1.err
timeout 600 python bench.py --config c3 --no-cpu > $O/bench_c3.json 2> $O/bench_c3.err
APEX_LIB=ab/v1.so timeout 600 python bench.py --config c3 --no-cpu > $O/bench_c3_v1.json 2> $O/bench_c3_v1.err
