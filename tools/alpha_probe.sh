# C3/C2 throughput of the staged kernel vs the ghost-layout CSoA block size alpha
for a in ${@:-256 4096 65536 1073741824}; do
  LBMG_GHOST_ALPHA=$a timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3 alpha', $a, round(d['value']), d['roofline']['kernel_ms'])"
  LBMG_GHOST_ALPHA=$a timeout 300 python bench.py --config c2 --steps 200 --warmup 5 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2 alpha', $a, round(d['value']), d['roofline']['kernel_ms'])"
  LBMG_GHOST_ALPHA=$a LBMG_GHOST_DBG=2 timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3 copy alpha', $a, round(d['value']), d['roofline']['kernel_ms'])"
done
