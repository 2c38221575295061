#!/bin/bash
# timing-only A/B of prebuilt library variants:  tools/ab3.sh "<ops>" "<configs>" var1 var2 ...
ops=$1; shift
cfgs=$1; shift
for v in "$@"; do
  if [ "$v" = base ]; then lib=$PWD/paper_2408_11971_b200/_lib/libhsz_b200.so
  else lib=$PWD/paper_2408_11971_b200/_lib/var_$v.so; fi
  export HSZ_NO_BUILD=1 HSZ_B200_LIB=$lib
  for c in $cfgs; do
    echo "$v config$c $(timeout 300 python tools/time_ops.py --config $c --reps 20 --ops $ops 2>&1 | tail -1)"
  done
done
