#!/bin/bash
# Per-launch durations of SENT 512^2 elastic GMG-PCG solves, next to the unprofiled wall time per
# solve (graph mode and eager): the gap between the two is launch/dependency overhead.
O=gpurun_out/vc
mkdir -p $O
python tools/el_time.py 512 > $O/el_time.txt 2>&1 || exit 1
TAG=eager PF_NO_GRAPHS=1 python tools/el_time.py 512 >> $O/el_time.txt 2>&1 || exit 1
PF_NO_GRAPHS=1 REPS=1 ncu --clock-control none --cache-control none --metrics gpu__time_duration.sum --csv \
    --log-file $O/launches.csv python tools/el_time.py 512 > $O/el_time_ncu.txt 2>&1
python tools/ncu_launch_summary.py $O/launches.csv > $O/summary.txt
cat $O/el_time.txt $O/summary.txt
