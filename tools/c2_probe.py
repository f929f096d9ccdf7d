"""Fluid-kernel time of the C2 grid with and without the sphere (IB) and with
periodic x, to attribute C2's per-node cost (run on the GPU box)."""
import statistics
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2101_11856_b200 as lbm  # noqa: E402
from tests import scenes  # noqa: E402


def fluid_ms(cfg, steps=30):
    r = lbm.Runner(lbm.build_scene(cfg))
    r.advance(5)
    rows = []
    r.advance(steps, timings=rows)
    return statistics.mean(x.seconds for x in rows if x.phase == "fluid") * 1e3


base = scenes.sphere()
base.alpha = 1 << 22
print("c2 with sphere", fluid_ms(base))
nos = scenes.sphere()
nos.alpha = 1 << 22
nos.solids = []
print("c2 no solids", fluid_ms(nos))
per = scenes.sphere()
per.solids = []
per.faces = scenes.faces(*["periodic"] * 6)
print("c2 grid all periodic", fluid_ms(per))
big = scenes.channel(n=256, nz=256)
print("256^3 channel", fluid_ms(big), "per-node-equivalent for 4.19M:", fluid_ms(big) * 4194304 / 256 ** 3)
