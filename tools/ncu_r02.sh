#!/bin/bash
# Round-2 evidence: the headline bench line (driver arguments), the ncu launch list of the same
# command (eager Krylov loops: ncu cannot profile kernel nodes of graphs with conditional nodes),
# and full captures of the dominant kernels of the SENT 512^2 elastic solve (persistent coarse
# cycle, the fine smoother strips, the CG update) read back as raw CSV.
O=gpurun_out/r02
mkdir -p $O
python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
PF_NO_GRAPHS=1 ncu --clock-control none --metrics gpu__time_duration.sum -c 6000 --csv \
    --log-file $O/launches_sent512.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-e2e > $O/ncu_bench.log 2>&1
python tools/ncu_launch_summary.py $O/launches_sent512.csv > $O/launches_summary.txt
export PF_NO_GRAPHS=1 REPS=1
python tools/el_time.py 512 > $O/el_time.log 2>&1
for k in k_gmg_coarse "OpKuuILb0ELi1E" "OpKuuILb0ELi2E" k_cg_update_gmg; do
  tag=$(echo "$k" | tr -dc 'A-Za-z0-9_')
  ncu --clock-control none --set full --import-source on --kernel-name-base mangled -k "regex:$k" -s 3 -c 1 \
      -o $O/sent_$tag python tools/el_time.py 512 > $O/sent_$tag.log 2>&1
  ncu -i $O/sent_$tag.ncu-rep --page raw --csv > $O/sent_$tag.raw.csv 2>/dev/null
done
ls -la $O
