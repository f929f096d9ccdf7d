# per-direction array stride padding (units of 256 slots) vs fluid kernel time, C2 and C3
for pd in ${@:-0 1 2 3 8 17}; do
LBMG_A_PAD=$pd timeout 300 python bench.py --config c2 --steps 200 --warmup 5 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pad', $pd, 'c2', round(d['value']), d['roofline']['kernel_ms'])"
LBMG_A_PAD=$pd timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pad', $pd, 'c3', round(d['value']), d['roofline']['kernel_ms'])"
done
