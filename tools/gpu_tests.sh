#!/bin/bash
# Run the -m gpu suite file by file, each under its own timeout, so one hang
# cannot hide the rest (run under gpurun from the repo root).
#   tools/gpu_tests.sh [per-file timeout s] [files...]
to=${1:-600}; shift
files=${@:-tests/test_gpu_*.py}
mkdir -p gpurun_out/tests
for f in $files; do
  b=$(basename $f .py)
  timeout $to python -m pytest $f -q -m gpu -p no:cacheprovider -x > gpurun_out/tests/$b.log 2>&1
  rc=$?
  echo "$b rc=$rc $(tail -1 gpurun_out/tests/$b.log)"
done
