#!/bin/bash
# A/B of prebuilt library variants (run under gpurun from the repo root).
#   tools/ab.sh "<ops>" "<configs>" var1 var2 ...
# each variant is paper_2408_11971_b200/_lib/var_<name>.so (built locally by
# tools/build_variant.sh); "base" = the default library.  For every variant:
# the GPU parity tests that cover the timed ops, then per-op device times.
ops=$1; shift
cfgs=$1; shift
mkdir -p gpurun_out/ab
for v in "$@"; do
  if [ "$v" = base ]; then lib=$PWD/paper_2408_11971_b200/_lib/libhsz_b200.so
  else lib=$PWD/paper_2408_11971_b200/_lib/var_$v.so; fi
  export HSZ_NO_BUILD=1 HSZ_B200_LIB=$lib
  timeout 600 python -m pytest -q -m gpu -p no:cacheprovider -x tests/test_gpu_paths.py tests/test_gpu_parity.py \
     tests/test_gpu_configs.py -k "scalar_mul or chain or config or smul or random" > gpurun_out/ab/$v.pytest.log 2>&1
  echo "$v parity rc=$? $(tail -1 gpurun_out/ab/$v.pytest.log)"
  for c in $cfgs; do
    echo "$v config$c $(timeout 300 python tools/time_ops.py --config $c --reps 20 --ops $ops 2>&1 | tail -1)"
  done
done
