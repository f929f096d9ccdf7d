OUT=gpurun_out; mkdir -p $OUT; T=${1:-pf}
timeout 300 python tools/iter/oh.py > $OUT/overhead_$T.log 2>&1
timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > $OUT/bench_c2_$T.json 2>&1
LBMG_GHOST_DBG=16 timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > $OUT/bench_c2_spf_$T.json 2>&1
timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > $OUT/bench_c2b_$T.json 2>&1
LBMG_GHOST_DBG=16 timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > $OUT/bench_c2b_spf_$T.json 2>&1
