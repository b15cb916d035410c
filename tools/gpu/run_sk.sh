set -u
O=gpurun_out/sk1; mkdir -p $O
timeout 600 python -m pytest tests/test_decode_gpu.py -q -m gpu -k "streamk or ring or split_inv" > $O/pytest.log 2>&1; echo "pytest rc=$?"
for c in c3 c4 c2 c5; do
timeout 900 python tools/tune.py --config $c --chunks 0 --reps 15 --scheds=-1,0,20,50,100,200,-1,0,20,50,100,200 > $O/tune_$c.log 2>&1; echo "tune $c rc=$?"
done
