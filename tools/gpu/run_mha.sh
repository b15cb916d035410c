set -u
O=gpurun_out/mha; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu -x -k "f16 or sanitizer or c2 or random or churn" > $O/pytest.log 2>&1; echo "pytest rc=$?"
for r in 1 2; do for lib in mha_simt mha_mma; do
APEX_LIB=ab/$lib.so timeout 600 python tools/tune.py --config c2 --chunks 0 --reps 20 | grep '^{"grid' | sed "s/^/$lib /" >> $O/tune_c2.log
done; done
for lib in mha_simt mha_mma; do
APEX_LIB=ab/$lib.so timeout 600 python bench.py --config c2 --no-cpu --no-e2e > $O/bench_c2_$lib.json 2>/dev/null
APEX_LIB=ab/$lib.so timeout 600 python tools/latency_probe.py --shape f16,32,32,8,1024 | sed "s/^/$lib /" >> $O/lat.log
done
