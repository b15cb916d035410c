set -u
O=gpurun_out/guided; mkdir -p $O
timeout 600 python -m pytest tests/test_decode_gpu.py -q -m gpu -k "streamk" > $O/pytest.log 2>&1; echo "pytest rc=$?"
S=-1,-2:8/800/900/950,-2:16/800/900/950,-2:6/700/850/950,-2:8/900/950/980,-2:12/850/930/970,-2:4/600/800/920
for c in c3 c4 c2 c5; do
timeout 900 python tools/tune.py --config $c --chunks 0 --reps 15 --scheds=$S,$S > $O/tune_$c.log 2>&1; echo "tune $c rc=$?"
done
