set -u
O=gpurun_out/ncu_lat; mkdir -p $O
APEX_LIB=ab/v1.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:apex_decode_kernel -s 5 -c 1 -o $O/lat_b1_16k python tools/latency_probe.py --shape bf16,32,8,1,16384 --reps 3 > $O/lat_b1_16k.log 2>&1
APEX_LIB=ab/v1.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:apex_decode_kernel -s 5 -c 1 -o $O/lat_c1 python tools/latency_probe.py --shape f32,32,32,1,512 --reps 3 > $O/lat_c1.log 2>&1
APEX_LIB=ab/v1.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:apex_ -s 10 -c 2 -o $O/lat_b1_64k python tools/latency_probe.py --shape bf16,32,8,1,65536 --reps 3 > $O/lat_b1_64k.log 2>&1
echo done
