import sys, os
sys.path.insert(0, os.getcwd())
import paper_2101_11856_b200 as lbm
from tests import scenes
which = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = scenes.sphere() if which == "c2" else scenes.channel(n=512)
cfg.alpha = 1 << 30
r = lbm.Runner(lbm.build_scene(cfg))
r.advance(int(sys.argv[2]) if len(sys.argv) > 2 else 16)
