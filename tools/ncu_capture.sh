#!/bin/bash
# ncu evidence for profiles/ (run on the GPU box from the repo root; each capture after the same
# command has exited 0 without ncu).  Outputs land in gpurun_out/ncu/.
set -u
O=gpurun_out/ncu
mkdir -p $O
N="ncu --clock-control none"
# 1) launch list (per-launch gpu__time_duration) of the headline bench command
python bench.py --steps 2 --warmup 1 --no-sweep --no-e2e > $O/bench_plain.json 2>/dev/null && \
$N --metrics gpu__time_duration.sum -c 4000 --csv --log-file $O/launches_sent512.csv \
    python bench.py --steps 2 --warmup 1 --no-sweep --no-e2e > /dev/null 2>&1
# 2) full captures of the SENT kernels inside one GMG-PCG elastic solve (512^2 crossed)
python tools/gmg_prof.py 512 2 > /dev/null 2>&1 && for k in "OpKuu<0, 1>" "OpKuu<0, 2>" "OpKuu<0, 3>" "OpKuu<0, 4>" "OpKuu<1, 0>" "k_cg_update_gmg" "k_pre_first" "k_gmg_tail"; do
  tag=$(echo "$k" | tr -dc 'A-Za-z0-9_')
  $N --set full --import-source on --kernel-name-base demangled -k "regex:$k" -s 2 -c 1 \
     -o $O/sent_$tag python tools/gmg_prof.py 512 2 > /dev/null 2>&1
  ncu -i $O/sent_$tag.ncu-rep --page raw --csv > $O/sent_$tag.raw.csv 2>/dev/null
  [ "$tag" = "OpKuu01" ] || rm -f $O/sent_$tag.ncu-rep
done
# 3) operator applies at config-5 sizes
for spec in "Kuu 8192 union_jack" "Kuu 8192 crossed" "Kaa 8192 crossed" "Kuu 256 kuhn6" "Kaa 256 kuhn6"; do
  set -- $spec
  python tools/opbench.py $1 $2 $3 3 > $O/op_$1_$2_$3.txt 2>&1 && \
  $N --set full --import-source on -k regex:k_strip -s 2 -c 1 -o $O/op_$1_$2_$3 python tools/opbench.py $1 $2 $3 3 > /dev/null 2>&1
  ncu -i $O/op_$1_$2_$3.ncu-rep --page raw --csv > $O/op_$1_$2_$3.raw.csv 2>/dev/null
  rm -f $O/op_$1_$2_$3.ncu-rep
done
du -sh $O
ls -la $O
