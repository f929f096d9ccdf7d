import sys, os, statistics, json
sys.path.insert(0, os.getcwd())
import paper_2101_11856_b200 as lbm
from tests import scenes
cfg = scenes.city_c4(); cfg.alpha = 1 << 30
r = lbm.Runner(lbm.build_scene(cfg))
r.advance(3)
rows = []
r.advance(6, timings=rows)
ib = statistics.mean(x.seconds for x in rows if x.phase == "ib")
fl = statistics.mean(x.seconds for x in rows if x.phase == "fluid")
t = r.measure_cost(r.block_edge(), r.alpha(), 1, 6)
print(json.dumps({"scatter": os.environ.get("LBMG_IB_SCATTER", "smem"), "ms_per_step": t * 1e3, "ib_ms": ib * 1e3, "fluid_ms": fl * 1e3,
                  "GLUPS": 252e6 / t / 1e9}), flush=True)
