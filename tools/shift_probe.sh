for sh in 0 4 16 64 128; do for m in 0 2; do d=$(( sh * 256 + m ));
LBMG_GHOST_DBG=$d timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('shift', $sh, 'mode', $m, round(d['value']), d['roofline']['kernel_ms'])"; done; done
