set -u
O=gpurun_out/ab1; mkdir -p $O
for r in 1 2; do for lib in base noepi; do
APEX_LIB=ab/$lib.so timeout 600 python tools/tune.py --config c3 --chunks 0 --reps 15 --scheds=-2:8/900/950/980,-2:16/900/950/980,-2:32/900/950/980 | grep '^{"grid' | sed "s/^/$lib /" >> $O/tune_c3.log
done; done
