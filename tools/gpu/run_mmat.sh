set -u
O=gpurun_out/mmat; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest.log 2>&1; echo "pytest rc=$?"
for c in c3 c4 c5; do
for r in 1 2; do for lib in mmaold mmat; do
APEX_LIB=ab/$lib.so timeout 600 python tools/tune.py --config $c --chunks 0 --reps 20 | grep '^{"grid' | sed "s/^/$lib /" >> $O/tune_$c.log
done; done; done
for lib in mmaold mmat; do
APEX_LIB=ab/$lib.so timeout 600 python bench.py --config c3 --no-cpu --no-e2e > $O/bench_c3_$lib.json 2>/dev/null
done
