#!/bin/bash
# Warm-cache per-launch durations of SENT 512^2 elastic GMG-PCG solves (graph mode), next to the
# unprofiled wall time per solve: the gap between the two is launch/dependency overhead.
O=gpurun_out/vc
mkdir -p $O

python tools/el_time.py 512 > $O/el_time.txt 2>&1 || exit 1
REPS=2 ncu --clock-control none --cache-control none --metrics gpu__time_duration.sum --csv \
    --log-file $O/launches.csv python tools/el_time.py 512 > $O/el_time_ncu.txt 2>&1
python tools/ncu_launch_summary.py $O/launches.csv > $O/summary.txt
cat $O/el_time.txt $O/summary.txt
