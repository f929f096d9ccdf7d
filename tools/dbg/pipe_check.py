"""Quick pipeline check: step pipeline (fluid variant 2) vs the per-kernel
staged path (variant 0) on a few scenes, then C2 timing of both."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2101_11856_b200 as lbm
from tests import scenes

def run(cfg, steps, variant):
    r = lbm.Runner(lbm.build_scene(cfg))
    if r.variant()[0] != variant:
        r.set_variant(variant, 0)
    st = r.advance(steps)
    return r, st

for name, cfg, steps in [("cavity20", scenes.cavity(n=20), 37), ("chan", scenes.channel(n=24, nz=30), 23),
                         ("mix", scenes.outflow_mix(12, 8, 10), 19),
                         ("sphere", scenes.sphere(48, 32, 32, center=(16, 16, 16), radius=5.0, subdiv=3, r=0.6), 21),
                         ("fins", scenes.rotating_fins(96, 48, 48), 17)]:
    a, sa = run(cfg, steps, 2)
    b, sb = run(cfg, steps, 0)
    fa, fb = a.gather_f(), b.gather_f()
    print(name, "variant", a.variant(), sa.ok, sb.ok, a.step_count(), b.step_count(), "max|df|", np.abs(fa - fb).max(),
          "rho", np.abs(a.gather_rho() - b.gather_rho()).max(), flush=True)

cfg = scenes.sphere(); cfg.alpha = 1 << 22
for v in (2, 0):
    r = lbm.Runner(lbm.build_scene(cfg))
    if r.variant()[0] != v: r.set_variant(v, 0)
    r.advance(20)
    import ctypes
    for k in (40, 200):
        t = r.measure_cost(r.block_edge(), r.alpha(), 2, k)
        print("C2 variant", v, "steps", k, "ms/step %.4f" % (t * 1e3), "GLUPS %.2f" % (4194304 / t / 1e9), flush=True)
