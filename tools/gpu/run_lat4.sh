set -u
O=gpurun_out/lat4; mkdir -p $O
timeout 600 python tools/latency_probe.py > $O/lat.log
for sh in bf16,32,8,32,2048 bf16,32,8,128,512 bf16,32,8,64,2048 bf16,32,8,128,1024 bf16,32,8,16,16384 bf16,32,8,256,512 bf16,32,8,64,4096 bf16,32,8,128,2048; do
for lt in 512 1024; do
APEX_LAT_TILES=$lt timeout 600 python tools/latency_probe.py --shape $sh | sed "s/^/lat$lt /" >> $O/lat2.log
done; done
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?"
