OUT=gpurun_out; mkdir -p $OUT; T=${1:-cf8}
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_$T.log 2>&1; echo "pytest_exit=$?" >> $OUT/pytest_$T.log
timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > $OUT/bench_c2_$T.json 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_c2d_$T.json 2>&1
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c4_$T.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 150 --csv --log-file $OUT/launches_c2_$T.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
