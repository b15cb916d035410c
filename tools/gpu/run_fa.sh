set -u
O=gpurun_out/fa; mkdir -p $O
timeout 900 python -m pytest tests/test_fused_append_gpu.py tests/test_decode_gpu.py -q -m gpu -x -k "fused or sanitizer or ragged" > $O/pytest.log 2>&1; echo "pytest rc=$?"
