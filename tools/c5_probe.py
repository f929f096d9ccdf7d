"""configs[4] on ONE B200: rotating fan (fin comb about the domain's x axis,
one revolution per 500 steps) in a 512x256x256 box: the moving-solid IB
stress case.  Prints one JSON line per IB variant (fused / split)."""
import json
import math
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2101_11856_b200 as lbm  # noqa: E402
from tests import scenes  # noqa: E402


def fan_c5(r=0.5):
    cfg = scenes.acm(lbm.SceneConfig(nx=512, ny=256, nz=256, viscosity=0.02))
    cfg.faces = scenes.faces(*["no-slip"] * 6)
    cfg.solids = [lbm.SolidConfig(lbm.MeshConfig(type="fin-comb", origin=(208, 88, 88), fins=8, fin_length=80,
                                                 fin_height=64, fin_spacing=10.0), poisson_radius=r,
                                  # one revolution per 2000 steps: tip speed ~0.25 at this 4x twin scale
                                  motion=lbm.RigidMotion(angular_velocity=(2 * math.pi / 2000, 0, 0),
                                                         center=(248, 123, 120)))]
    cfg.block_edge = 2
    cfg.alpha = 1 << 30
    return cfg


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    cfg = fan_c5()
    scene = lbm.build_scene(cfg)
    ns = len(scene.samples(0)["source_id"])
    r = lbm.Runner(scene)
    n = cfg.nx * cfg.ny * cfg.nz
    for v in ((0, 0), (0, 1)):
        r.set_variant(*v)
        st = r.advance(3)
        if not st.ok:
            print(json.dumps({"variant": v, "diverged": True, "step": st.step}), flush=True)
            return
        rows = []
        r.advance(steps, timings=rows)
        ib = statistics.mean(x.seconds for x in rows if x.phase == "ib")
        fl = statistics.mean(x.seconds for x in rows if x.phase == "fluid")
        sec = r.measure_cost(r.block_edge(), r.alpha(), 1, steps)
        print(json.dumps({"workload": "configs[4] rotating fan 512x256x256 on 1 GPU", "variant": v, "samples": ns,
                          "moving": True, "ms_per_step": sec * 1e3, "MLUPS": n / sec / 1e6, "ib_ms": ib * 1e3,
                          "fluid_ms": fl * 1e3, "step": r.step_count()}), flush=True)


if __name__ == "__main__":
    main()
