#!/bin/bash
# Round measurement on one B200: parity suite, bench lines (C2 headline with
# CPU baseline, C3), launch lists, one full ncu capture of the fluid kernel
# per config and of the C2 boundary/IB kernels.  Usage: bash tools/gpu_round.sh <tag>
TAG=${1:-r}
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu_$TAG.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_$TAG.log 2>&1; echo "pytest_exit=$?" >> $OUT/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1
timeout 600 python bench.py --steps 200 --warmup 5 > $OUT/bench_c2_$TAG.json 2> $OUT/bench_c2_$TAG.err
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c3_$TAG.json 2> $OUT/bench_c3_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 150 --csv \
   --log-file $OUT/launches_c2_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
   --log-file $OUT/launches_c3_$TAG.csv python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fluid_ghost|ghost_fill|ib_fused" -s 9 -c 3 \
   -o $OUT/prof_c2_$TAG python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fluid_ghost -s 3 -c 1 \
   -o $OUT/prof_c3_$TAG python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la $OUT
gzip -f $OUT/*.ncu-rep; ls -la $OUT
