#!/bin/bash
# Round measurement on one B200 (run under gpurun from the repo root):
#   bash tools/gpu_round.sh <tag> [tests] [bench] [ncu] [big]
# tests: pytest -m gpu + smoke; bench: C2 (driver settings and 200 steps) and
# C3 lines; big: C4 and C5 lines; ncu: launch lists + full captures.
TAG=${1:-r}; shift
WHAT=${*:-tests bench}
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu_$TAG.txt 2>&1
has() { [[ " $WHAT " == *" $1 "* ]]; }
if has tests; then
  timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > $OUT/pytest_$TAG.log 2>&1; echo "pytest_exit=$?" >> $OUT/pytest_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1
fi
if has bench; then
  timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench_c2d_$TAG.json 2> $OUT/bench_c2d_$TAG.err
  timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > $OUT/bench_c2_$TAG.json 2> $OUT/bench_c2_$TAG.err
  timeout 600 python bench.py --config c3 --steps 20 --warmup 3 > $OUT/bench_c3_$TAG.json 2> $OUT/bench_c3_$TAG.err
  timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
fi
if has big; then
  timeout 900 python bench.py --config c4 --steps 10 --warmup 3 > $OUT/bench_c4_$TAG.json 2> $OUT/bench_c4_$TAG.err
  timeout 900 python bench.py --config c5 --steps 40 --warmup 5 > $OUT/bench_c5_$TAG.json 2> $OUT/bench_c5_$TAG.err
fi
if has ncu; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 150 --csv \
     --log-file $OUT/launches_c2_$TAG.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
     --log-file $OUT/launches_c3_$TAG.csv python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fluid_ghost|ghost_fill|ib_fused" -s 9 -c 3 \
     -o $OUT/prof_c2_$TAG python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fluid_ghost|ghost_fill" -s 3 -c 2 \
     -o $OUT/prof_c3_$TAG python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  gzip -f $OUT/*.ncu-rep
fi
ls -la $OUT | tail -30
if has ibprof; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ib_fused|ib_band_moments" -s 2 -c 2 \
     -o $OUT/prof_c4ib_$TAG python bench.py --config c4 --steps 1 --warmup 2 --no-cpu-baseline > /dev/null 2>&1
  gzip -f $OUT/*.ncu-rep
fi
