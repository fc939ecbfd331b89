#!/bin/bash
# ncu --set full capture of the persistent damage PCG on its free strips: three launches in schedule
# step 16 of the config-3 slab (the step in which the cracks form).  Run on the GPU box from the repo
# root (after the same command has exited 0 without ncu); outputs in gpurun_out/ncu_pcg/, summary
# copied to profiles/r02z_ncu_pcg_sparse/.
set -u
O=gpurun_out/ncu_pcg
mkdir -p $O
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_pcg_kaa --launch-skip 200 --launch-count 3 \
  -o $O/pcg_kaa_thermal python tools/sent_window.py --workload thermal --n 512 --steps 17 --no-split \
  --out $O/window_ncu.json > $O/ncu.log 2>&1
tail -3 $O/ncu.log
ncu -i $O/pcg_kaa_thermal.ncu-rep --page raw --csv > $O/pcg_kaa_thermal.raw.csv 2>/dev/null
python tools/ncu_summary.py $O/summary.json $O/pcg_kaa_thermal.raw.csv
ls -la $O
