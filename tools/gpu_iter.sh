#!/bin/bash
# Iteration run on one B200: GPU parity suite, C2 (200 steps) / C3 / C4 bench
# lines and the C2 launch list.  Usage: bash tools/gpu_iter.sh <tag> [notests] [noc4]
TAG=${1:-i}; shift
OUT=gpurun_out; mkdir -p $OUT
has() { local k=$1; shift; [[ " $* " == *" $k "* ]]; }
if ! has notests "$@"; then
  timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/pytest_$TAG.log 2>&1; echo "pytest_exit=$?" >> $OUT/pytest_$TAG.log
fi
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > $OUT/bench_c2_$TAG.json 2> $OUT/bench_c2_$TAG.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_c2d_$TAG.json 2> $OUT/bench_c2d_$TAG.err
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c3_$TAG.json 2> $OUT/bench_c3_$TAG.err
if ! has noc4 "$@"; then
  timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c4_$TAG.json 2> $OUT/bench_c4_$TAG.err
  timeout 900 python bench.py --config c5 --steps 40 --warmup 5 --no-cpu-baseline > $OUT/bench_c5_$TAG.json 2> $OUT/bench_c5_$TAG.err
fi
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 150 --csv \
   --log-file $OUT/launches_c2_$TAG.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
ls -la $OUT | tail -12
