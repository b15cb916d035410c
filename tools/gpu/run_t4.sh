set -u
O=gpurun_out/t4; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?"
