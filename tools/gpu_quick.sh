#!/bin/bash
# Quick check on one B200: the GPU parity suite, C2/C3 bench lines and the C2
# launch list.  Usage: bash tools/gpu_quick.sh <tag>
TAG=${1:-q}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_$TAG.log 2>&1; echo "pytest_exit=$?" >> $OUT/pytest_$TAG.log
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > $OUT/bench_c2_$TAG.json 2> $OUT/bench_c2_$TAG.err
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c3_$TAG.json 2> $OUT/bench_c3_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 150 --csv \
   --log-file $OUT/launches_c2_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
# CTA-size probe of the staged fluid kernel on C2 (LBMG_GHOST_THREADS), on request
for T in ${PROBE_T:-}; do
  LBMG_GHOST_THREADS=$T timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > $OUT/bench_c2_T${T}_$TAG.json 2>&1
done
