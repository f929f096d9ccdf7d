import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2101_11856_b200 as lbm
from tests import scenes
cfg = scenes.sphere(48, 32, 32, center=(16, 16, 16), radius=5.0, subdiv=3, r=0.6)
for pre in (0, 1, 5):
    g = lbm.Runner(lbm.build_scene(cfg)); h = lbm.Runner(lbm.build_scene(cfg))
    if pre:
        g.advance(pre); h.advance(pre)
    c = g.clone()
    out = []
    for k in range(4):
        g.advance(1); c.advance(1); h.advance(1)
        fg, fc, fh = g.gather_f(), c.gather_f(), h.gather_f()
        out.append((np.abs(fg - fc).max(), np.abs(fg - fh).max(), np.argmax(np.abs(fg-fc).max(axis=1))))
    print("pre", pre, out, flush=True)
