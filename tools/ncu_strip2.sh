#!/bin/bash
# ncu evidence for the v2 (TMA) 2D strip engine against the v1 (cp.async) engine: 8192^2 applies.
# Run on the GPU box from the repo root; outputs in gpurun_out/ncu2/.
set -u
O=gpurun_out/ncu2
mkdir -p $O
N="ncu --clock-control none"
for eng in 0 1; do
  for spec in "Kuu 8192 union_jack" "Kuu 8192 crossed" "Kaa 8192 union_jack"; do
    set -- $spec
    tag=v$((eng+1))_$1_$2_$3
    PF_STRIP2=$eng python tools/opbench.py $1 $2 $3 5 > $O/$tag.txt 2>&1 && \
    PF_STRIP2=$eng $N --set full --import-source on -k regex:k_strip2 -s 2 -c 1 -o $O/$tag python tools/opbench.py $1 $2 $3 3 > /dev/null 2>&1
    ncu -i $O/$tag.ncu-rep --page raw --csv > $O/$tag.raw.csv 2>/dev/null
    [ "$tag" = "v2_Kuu_8192_union_jack" ] || rm -f $O/$tag.ncu-rep
  done
done
ls -la $O
