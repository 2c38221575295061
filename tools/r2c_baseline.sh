#!/bin/bash
# HEAD verification run: per-file GPU tests, the default bench line, one ncu --set full capture (config 4)
set -u
tag=${1:-r2c}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > $out/gpu.txt 2>&1
tools/gpu_tests.sh 900 > $out/tests_summary.txt 2>&1
cat $out/tests_summary.txt
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err
echo "bench rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"compress_f32|recode_kernel|decode_pipe" -c 5 \
    -o $out/full python tools/prof_ops.py --config 4 --reps 1 > $out/ncu_full.log 2>&1
echo "ncu full rc=$?"
ls -la $out
