#!/bin/bash
# One GPU session: bench lines + ncu launch list + full ncu captures of the
# hot kernels.  Outputs land in gpurun_out/ (summaries get copied to
# profiles/).  Usage (from the repo root, under gpurun):
#   bash tools/gpu_bench_profile.sh <tag> [--no-ncu]
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu_$TAG.txt 2>&1
timeout 600 python bench.py --steps 100 --warmup 5 > $OUT/bench_c2_$TAG.json 2> $OUT/bench_c2_$TAG.err
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c3_$TAG.json 2> $OUT/bench_c3_$TAG.err
LBMG_BULK_MINB=4 timeout 600 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c3_minb4_$TAG.json 2> $OUT/bench_c3_minb4_$TAG.err
if [ "$2" == "--no-ncu" ]; then exit 0; fi
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv \
   --log-file $OUT/launches_c2_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2> $OUT/ncu_launch_$TAG.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fluid_bulk|fluid_shell|ib_spread" -s 12 -c 3 \
   -o $OUT/prof_c2_$TAG python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2> $OUT/ncu_full_$TAG.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fluid_bulk -s 3 -c 1 \
   -o $OUT/prof_c3_$TAG python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2> $OUT/ncu_full_c3_$TAG.err
ls -la $OUT
