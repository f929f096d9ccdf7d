import sys, os
sys.path.insert(0, os.getcwd())
import paper_2101_11856_b200 as lbm
from tests import scenes
which = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = scenes.sphere() if which == "c2" else scenes.channel(n=512)
cfg.alpha = 1 << 30
r = lbm.Runner(lbm.build_scene(cfg))
r.advance(10)
n = cfg.nx * cfg.ny * cfg.nz
t = r.measure_cost(r.block_edge(), r.alpha(), 2, 40 if which == "c2" else 8)
print(which, os.environ.get("LBMG_PIPE_DBG", "0"), os.environ.get("LBMG_PIPELINE", "1"), "ms/step %.4f GLUPS %.2f" % (t * 1e3, n / t / 1e9), flush=True)
