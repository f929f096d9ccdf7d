#!/bin/bash
# Quick GPU iteration: parity suite + C2/C3 bench lines (+ optional A/B env).
# Usage under gpurun: bash tools/gpu_check.sh <tag> [extra bench env, e.g. LBMG_BULK=ldg]
TAG=${1:-x}; shift
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_$TAG.log 2>&1; echo "pytest_exit=$?" >> $OUT/pytest_$TAG.log
tail -3 $OUT/pytest_$TAG.log
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > $OUT/bench_c2_$TAG.json 2> $OUT/bench_c2_$TAG.err
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c3_$TAG.json 2> $OUT/bench_c3_$TAG.err
for v in "$@"; do
  env $v timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > $OUT/bench_c2_${TAG}_$v.json 2>&1
  env $v timeout 600 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c3_${TAG}_$v.json 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["value"]), d["roofline"]["frac"] if d.get("roofline") else None, d["ms_per_step"])
    except Exception as e: print(f, "ERR", e)
PY
if [ -n "$NCU" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:fluid_bulk -s 3 -c 1 \
     -o $OUT/prof_c3_$TAG python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2> $OUT/ncu_c3_$TAG.err
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fluid_" -s 6 -c 2 \
     -o $OUT/prof_c2_$TAG python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2> $OUT/ncu_c2_$TAG.err
fi
