set -u
O=gpurun_out/tlb; mkdir -p $O
for L in 1 32 1 32; do
timeout 600 python tools/tune.py --config c3 --chunks 0 --reps 64 --layers $L | grep '^{"grid' | sed "s/^/L$L /" >> $O/tune.log
done
