#!/bin/bash
# Bench + ncu evidence for profiles/ (run under gpurun from the repo root).
#   tools/round_profile.sh <tag>
set -u
tag=${1:-snap}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > $out/gpu.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench.json 2> $out/bench.err
echo "bench rc=$?"
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $out/bench_short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \
    --clock-control none --csv --log-file $out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $out/ncu_launches.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"encode_kernel|decode_kernel|moments_kernel" \
    -c 4 -o $out/full python tools/prof_ops.py --reps 1 > $out/ncu_full.log 2>&1
echo "ncu full rc=$?"
