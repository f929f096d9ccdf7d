"""Small ghost-layout runs for compute-sanitizer (memcheck / racecheck / synccheck):
    compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2101_11856_b200 as lbm  # noqa: E402
from tests import scenes  # noqa: E402

runs = [
    ("cavity", scenes.cavity(n=24), 1),
    ("sphere", scenes.sphere(48, 32, 32, center=(16, 16, 16), radius=5.0, subdiv=3, r=0.6), 1),
    ("edge-mix x2 regions", scenes.outflow_mix(12, 8, 10), 2),
    ("channel periodic", scenes.channel(n=16, nz=20), 1),
]
for name, cfg, regions in runs:
    r = lbm.Runner(lbm.build_scene(cfg), regions=regions)
    st = r.advance(6)
    r.snapshot_begin()
    r.advance(2)
    t, rho, u = r.snapshot_wait()
    f = r.gather_f()
    print(name, st.ok, r.step_count(), float(rho.sum()), float(f.sum()))
