#!/bin/bash
# Round-2 evidence run (under gpurun, from the repo root):
#   tools/round2_profile.sh <tag>
# gpu tests, the default bench line (config 4 + config5_n1), the reference
# arm, the ncu launch list of the bench command and one ncu --set full
# capture of the hot kernels on config 4 (traffic for roofline.traffic).
set -u
tag=${1:-r2}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > $out/gpu.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider -rf > $out/pytest.log 2>&1
echo "pytest rc=$? $(tail -1 $out/pytest.log)"
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err
echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $out/reference.json 2> $out/reference.err
echo "reference rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -c 600 --csv --log-file $out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-scale-baseline > $out/ncu_launches.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"compress_f32|recode_kernel|decode_pipe|negate32|sadd_kernel|minmax_f32" -c 8 \
    -o $out/full python tools/prof_ops.py --config 4 --reps 1 > $out/ncu_full.log 2>&1
echo "ncu full rc=$?"
