set -u
O=gpurun_out/lat3; mkdir -p $O
timeout 600 python tools/latency_probe.py | sed "s/^/lat128 /" >> $O/lat.log
for sh in bf16,32,8,32,2048 bf16,32,8,128,512 bf16,32,8,64,2048 bf16,32,8,128,1024 bf16,32,8,16,16384 bf16,32,8,256,512; do
for lt in 128 256 512; do
APEX_LAT_TILES=$lt timeout 600 python tools/latency_probe.py --shape $sh | sed "s/^/lat$lt /" >> $O/lat.log
done; done
timeout 900 python -m pytest tests -q -m gpu -x -k "decode or graph or fused or config" > $O/pytest.log 2>&1; echo "pytest rc=$?"
