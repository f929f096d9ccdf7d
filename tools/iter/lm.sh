OUT=gpurun_out; mkdir -p $OUT; T=${1:-lm}
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_$T.log 2>&1; echo "pytest_exit=$?" >> $OUT/pytest_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$T.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_c2d_$T.json 2>&1
timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > $OUT/bench_c2_$T.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fluid_ghost" -s 3 -c 1 \
     -o $OUT/prof_c4_$T python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
gzip -f $OUT/*.ncu-rep
