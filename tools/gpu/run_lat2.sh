set -u
O=gpurun_out/lat2; mkdir -p $O
for lt in 64 128 256; do
APEX_LAT_TILES=$lt timeout 600 python tools/latency_probe.py | sed "s/^/lat$lt /" >> $O/lat.log
done
for sh in bf16,32,8,32,2048 bf16,32,8,128,512 bf16,32,8,64,1024; do
for lt in 64 128; do
APEX_LAT_TILES=$lt timeout 600 python tools/latency_probe.py --shape $sh | sed "s/^/lat$lt /" >> $O/lat.log
done; done
