"""C2 step composition probe: step time (CUDA events over advance) for the
headline scene and variants without the sphere / with every face periodic,
and per-kernel times from the timing rows (serialised)."""
import sys, os, json, statistics
sys.path.insert(0, os.getcwd())
import paper_2101_11856_b200 as lbm
from tests import scenes

def run(name, cfg):
    cfg.alpha = 1 << 22
    r = lbm.Runner(lbm.build_scene(cfg))
    r.advance(10)
    t = min(r.measure_cost(r.block_edge(), r.alpha(), 2, 100) for _ in range(3))
    rows = []
    r.advance(20, timings=rows)
    ph = {p: statistics.mean(x.seconds for x in rows if x.phase == p) * 1e6 for p in ("boundary", "ib", "fluid")
          if any(x.phase == p for x in rows)}
    print(json.dumps({"case": name, "step_us": t * 1e6, **{k + "_us": v for k, v in ph.items()}}), flush=True)

run("c2", scenes.sphere())
cfg = scenes.sphere(); cfg.solids = []; run("c2_nosphere", cfg)
cfg = scenes.sphere(); cfg.solids = []; cfg.faces = scenes.faces(*["periodic"] * 6); run("c2_periodic", cfg)
