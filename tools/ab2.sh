#!/bin/bash
# A/B of prebuilt library variants with the whole encoder-side parity set.
#   tools/ab2.sh "<ops>" "<configs>" var1 var2 ...   ("base" = the default library)
ops=$1; shift
cfgs=$1; shift
mkdir -p gpurun_out/ab
for v in "$@"; do
  if [ "$v" = base ]; then lib=$PWD/paper_2408_11971_b200/_lib/libhsz_b200.so
  else lib=$PWD/paper_2408_11971_b200/_lib/var_$v.so; fi
  export HSZ_NO_BUILD=1 HSZ_B200_LIB=$lib
  timeout 900 python -m pytest -q -m gpu -p no:cacheprovider -x tests/test_gpu_paths.py tests/test_gpu_parity.py \
     tests/test_gpu_adversarial.py tests/test_gpu_elementwise.py tests/test_gpu_watchdog.py tests/test_gpu_stress.py \
     tests/test_gpu_configs.py > gpurun_out/ab/$v.pytest.log 2>&1
  echo "$v parity rc=$? $(tail -1 gpurun_out/ab/$v.pytest.log)"
  for c in $cfgs; do
    echo "$v config$c $(timeout 300 python tools/time_ops.py --config $c --reps 20 --ops $ops 2>&1 | tail -1)"
  done
done
