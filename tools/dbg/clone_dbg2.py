import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2101_11856_b200 as lbm
from tests import scenes
cfg = scenes.sphere(48, 32, 32, center=(16, 16, 16), radius=5.0, subdiv=3, r=0.6)
for adv in ((5, 7), (5, 2), (1, 2), (0, 2), (0, 9)):
    g = lbm.Runner(lbm.build_scene(cfg)); h = lbm.Runner(lbm.build_scene(cfg))
    if adv[0]:
        g.advance(adv[0]); h.advance(adv[0])
    c = g.clone()
    g.advance(adv[1]); c.advance(adv[1]); h.advance(adv[1])
    fg, fc, fh = g.gather_f(), c.gather_f(), h.gather_f()
    print(adv, "g-c", np.abs(fg - fc).max(), "g-h", np.abs(fg - fh).max(), "steps", g.step_count(), c.step_count(), flush=True)
