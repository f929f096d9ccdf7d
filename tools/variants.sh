#!/bin/bash
# Collision-form sweep (LBMG_FORM 0..2) on C3 (512^3) and C2, and the IB
# spread variant (global RED vs shared-memory hash) on C2.
OUT=gpurun_out; TAG=${1:-v}
for f in 2 0 1; do
  LBMG_FORM=$f timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/form_c3_${f}_$TAG.json 2>&1
  LBMG_FORM=$f timeout 300 python bench.py --config c2 --steps 100 --warmup 5 --no-cpu-baseline > $OUT/form_c2_${f}_$TAG.json 2>&1
done
LBMG_IB_SPREAD=smem timeout 300 python bench.py --config c2 --steps 100 --warmup 5 --no-cpu-baseline > $OUT/spread_smem_c2_$TAG.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv \
   --log-file $OUT/launches_c2_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2> $OUT/ncu_launch_$TAG.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fluid_bulk|fluid_shell|ib_spread|ib_mark" -s 16 -c 4 \
   -o $OUT/prof_c2_$TAG python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2> $OUT/ncu_full_$TAG.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fluid_bulk -s 3 -c 1 \
   -o $OUT/prof_c3_$TAG python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2> $OUT/ncu_full_c3_$TAG.err
