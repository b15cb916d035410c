set -u
O=gpurun_out/fa2; mkdir -p $O
timeout 900 python -m pytest tests/test_fused_append_gpu.py tests/test_graph_gpu.py tests/test_decode_gpu.py -q -m gpu -x -k "fused or sanitizer or graph" > $O/pytest.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --config c1 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 600 python bench.py --config c1 --append separate > $O/bench_c1_sep.json 2> $O/bench_c1_sep.err
timeout 600 python bench.py --config c3 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config c3 --append separate --no-cpu > $O/bench_c3_sep.json 2> $O/bench_c3_sep.err
