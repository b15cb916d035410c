set -u
O=gpurun_out/ab3; mkdir -p $O
for c in c3 c5; do
for r in 1 2; do for lib in v1 v2 v2serial v2nopf v2plain; do
APEX_LIB=ab/$lib.so timeout 600 python tools/tune.py --config $c --chunks 0 --reps 10 --scheds=-2,-1 | grep '^{"grid' | sed "s/^/$lib /" >> $O/tune_$c.log
done; done; done
