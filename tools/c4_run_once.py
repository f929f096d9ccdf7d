import sys; sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import c4_probe, paper_2101_11856_b200 as lbm
cfg = c4_probe.city_c4()
r = lbm.Runner(lbm.build_scene(cfg))
r.advance(4)
