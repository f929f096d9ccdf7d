# staged fluid kernel CTA size (128 / 256 threads) on C3 and C2, plus the copy probe
for t in ${@:-128 256 512}; do
LBMG_GHOST_THREADS=$t timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('T', $t, 'c3', round(d['value']), d['roofline']['kernel_ms'])"
LBMG_GHOST_THREADS=$t LBMG_GHOST_DBG=2 timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('T', $t, 'c3copy', round(d['value']), d['roofline']['kernel_ms'])"
LBMG_GHOST_THREADS=$t timeout 300 python bench.py --config c2 --steps 200 --warmup 5 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('T', $t, 'c2', round(d['value']), d['roofline']['kernel_ms'])"
done
