# ghost-fill variants: per-direction threads (default) vs per-node threads
for v in dir node; do for c in c2 c3; do
LBMG_FILL=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ghost_fill -c 4 --csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | grep ghost_fill | tail -1 | awk -F'","' -v v=$v -v c=$c '{print "fill", v, c, $NF}'
done; done
