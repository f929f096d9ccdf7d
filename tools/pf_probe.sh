# L2 prefetch distance (tile periods) of the staged fluid kernel: C3 and C2
for d in ${@:-0 1 2}; do
LBMG_L2_PREFETCH=$d timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pf', $d, 'c3', round(d['value']), d['roofline']['kernel_ms'])"
LBMG_L2_PREFETCH=$d timeout 300 python bench.py --config c2 --steps 200 --warmup 5 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pf', $d, 'c2', round(d['value']), d['roofline']['kernel_ms'])"
done
