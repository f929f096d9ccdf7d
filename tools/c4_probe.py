"""configs[3] on ONE B200: 1200x250x840 "smoke through complex architecture"
(a seeded city of box solids, Poisson r = 0.7, x- inlet / x+ outflow, ground
no-slip), the whole domain on one GPU (254 M slots x 2 x 108 B = 55 GB).
Times the fused and the split IB pipelines (the tuner's IB dimension) and
prints one JSON line per variant."""
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import paper_2101_11856_b200 as lbm  # noqa: E402
from tests import scenes  # noqa: E402


def city_c4(n_boxes=220, seed=7, r=0.7, nx=1200, ny=250, nz=840):
    cfg = scenes.acm(lbm.SceneConfig(nx=nx, ny=ny, nz=nz, viscosity=0.02))
    cfg.faces = scenes.faces("inlet", "outflow", "no-slip", "no-slip", "no-slip", "no-slip")
    cfg.init_velocity = (0.05, 0.0, 0.0)
    rng = np.random.default_rng(seed)
    cfg.solids = []
    # non-overlapping lots (overlapping boxes double the local sample density,
    # which the unnormalised penalty force does not survive)
    lots = [(150 + 50 * i, 20 + 50 * k) for i in range((nx - 300) // 50) for k in range((nz - 40) // 50)]
    for j in rng.permutation(len(lots))[:n_boxes]:
        lx, lz = lots[j]
        w, d = rng.uniform(10, 40, size=2)
        h = rng.uniform(20, 200)
        x0 = lx + rng.uniform(0, 45 - w)
        z0 = lz + rng.uniform(0, 45 - d)
        cfg.solids.append(lbm.SolidConfig(lbm.MeshConfig(type="box", lo=(x0, 1.2, z0), hi=(x0 + w, 1.2 + h, z0 + d)),
                                          poisson_radius=r))
    cfg.block_edge = 2
    cfg.alpha = 1 << 30
    return cfg


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    cfg = city_c4()
    t0 = time.time()
    scene = lbm.build_scene(cfg)
    t_build = time.time() - t0
    ns = sum(len(scene.samples(s)["source_id"]) for s in range(len(cfg.solids)))
    r = lbm.Runner(scene)
    n = cfg.nx * cfg.ny * cfg.nz
    for v in ((0, 0), (0, 1)):
        r.set_variant(*v)
        st = r.advance(3)
        if not st.ok:
            print(json.dumps({"variant": v, "diverged": True, "step": st.step, "reason": st.reason}), flush=True)
            return
        rows = []
        r.advance(steps, timings=rows)
        ib = statistics.mean(x.seconds for x in rows if x.phase == "ib")
        fl = statistics.mean(x.seconds for x in rows if x.phase == "fluid")
        bd = statistics.mean(x.seconds for x in rows if x.phase == "boundary")
        sec = r.measure_cost(r.block_edge(), r.alpha(), 1, steps)
        print(json.dumps({"workload": "configs[3] city 1200x250x840 on 1 GPU", "variant": v, "solids": len(cfg.solids),
                          "samples": ns, "scene_build_s": round(t_build, 2), "ok": st.ok,
                          "ms_per_step": sec * 1e3, "MLUPS": n / sec / 1e6, "ib_ms": ib * 1e3,
                          "fluid_ms": fl * 1e3, "boundary_ms": bd * 1e3}), flush=True)


if __name__ == "__main__":
    main()


def fluid_only(steps=5):
    cfg = city_c4()
    cfg.solids = []
    r = lbm.Runner(lbm.build_scene(cfg))
    r.advance(2)
    rows = []
    r.advance(steps, timings=rows)
    fl = statistics.mean(x.seconds for x in rows if x.phase == "fluid")
    print(json.dumps({"workload": "configs[3] grid without solids", "fluid_ms": fl * 1e3,
                      "kernel_TBps": 216 * cfg.nx * cfg.ny * cfg.nz / fl / 1e12}), flush=True)
