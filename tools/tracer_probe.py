"""Device tracer phase cost on the C2 sphere scene (run on the GPU box).

An emitter over most of the grid adds RATE particles per step; every
INTERVAL steps the per-phase CUDA-event timings of a few steps report the
tracer kernel time (emit + advect + retire, `tracers` row) against the live
cloud size.  Algorithmic bytes per live particle-step: 32 B read + 32 B
written (FP64 x, y, z + int64 birth) + 8 corners x 3 fp32 u* reads (96 B,
largely L2 hits for a dense cloud)."""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2101_11856_b200 as lbm  # noqa: E402
from tests import scenes  # noqa: E402

RATE = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
ROUNDS = int(sys.argv[2]) if len(sys.argv) > 2 else 5
INTERVAL = 100

cfg = scenes.sphere()
cfg.alpha = 1 << 22
cfg.emitters = [lbm.TracerEmitter(lo=(2.0, 4.0, 4.0), hi=(250.0, 123.0, 123.0), rate=RATE)]
r = lbm.Runner(lbm.build_scene(cfg))
for k in range(ROUNDS):
    assert r.advance(INTERVAL).ok
    rows = []
    r.advance(5, timings=rows)
    tr = statistics.mean(x.seconds for x in rows if x.phase == "tracers")
    fl = statistics.mean(x.seconds for x in rows if x.phase == "fluid")
    n = r.tracers().size()
    print(json.dumps({"step": r.step_count(), "live": n, "tracer_ms": tr * 1e3, "fluid_ms": fl * 1e3,
                      "ns_per_particle_step": tr * 1e9 / max(n, 1),
                      "gbs_64B": 64 * n / tr / 1e9 if tr > 0 else None}))
