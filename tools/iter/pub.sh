OUT=gpurun_out; mkdir -p $OUT; T=${1:-pub}
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_$T.log 2>&1; echo "pytest_exit=$?" >> $OUT/pytest_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$T.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 > $OUT/bench_c2d_$T.json 2> $OUT/bench_c2d_$T.err
timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > $OUT/bench_c2_$T.json 2>&1
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c4_$T.json 2>&1
timeout 600 python bench.py --config c5 --steps 40 --warmup 5 --no-cpu-baseline > $OUT/bench_c5_$T.json 2>&1
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c3_$T.json 2>&1
