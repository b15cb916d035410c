#!/bin/bash
# ncu evidence for the default bench (C5, N=1): timed-step launch list and one --set full
# capture of the decode kernel.  Outputs in gpurun_out/ncu/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/ncu; mkdir -p $O
python -m paper_2506_03296_b200.build > /dev/null
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_c5_timed.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > $O/launches_c5.out 2>&1
echo "launches rc=$?" >> $O/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:apex_decode_kernel -s 40 -c 1 \
  -o $O/prof_c5 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > $O/full_c5.out 2>&1
echo "full rc=$?" >> $O/rc.txt
ncu -i $O/prof_c5.ncu-rep --page raw --csv > $O/prof_c5_raw.csv 2>/dev/null
