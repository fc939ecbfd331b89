#!/bin/bash
# ncu --set full of the SENT 512^2 strip kernels inside one GMG-PCG elastic solve (mangled-name match)
O=gpurun_out/ncu
mkdir -p $O
python tools/gmg_prof.py 512 2 > /dev/null 2>&1 || exit 1
for k in OpKuuILb0ELi1E OpKuuILb0ELi2E OpKuuILb0ELi3E OpKuuILb0ELi4E OpKuuILb1ELi0E; do
  ncu --clock-control none --set full --import-source on --kernel-name-base mangled -k "regex:$k" -s 2 -c 1 \
      -o $O/sent_$k python tools/gmg_prof.py 512 2 > $O/sent_$k.log 2>&1
  ncu -i $O/sent_$k.ncu-rep --page raw --csv > $O/sent_$k.raw.csv 2>/dev/null
  [ "$k" = "OpKuuILb0ELi1E" ] && ncu -i $O/sent_$k.ncu-rep --page details --csv > $O/sent_$k.details.csv 2>/dev/null
  rm -f $O/sent_$k.ncu-rep
done
ls -la $O
