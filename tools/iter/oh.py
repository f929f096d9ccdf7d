"""Per-call overhead of Runner.advance(1) on a tiny grid (the e2e floor)."""
import sys, time
sys.path.insert(0, ".")
import paper_2101_11856_b200 as lbm
from tests import scenes
for name, cfg in (("cavity16", scenes.cavity(16)), ("sphere_small", scenes.sphere(32, 32, 32, center=(12, 16, 16), radius=4.0, subdiv=2, r=0.7))):
    r = lbm.Runner(lbm.build_scene(cfg))
    r.advance(20)
    n = 2000
    t0 = time.perf_counter()
    for _ in range(n):
        r.advance(1)
    dt = (time.perf_counter() - t0) / n
    t0 = time.perf_counter()
    r.advance(n)
    dt2 = (time.perf_counter() - t0) / n
    print(f"{name}: advance(1) per call {dt*1e6:.1f} us, advance({n}) per step {dt2*1e6:.1f} us", flush=True)
