"""Regenerate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref,
built from /root/reference/proj/src).  Run in the build container:

    make -C oracle ref && python tests/golden/make_golden.py

Fixtures (small, FP64, reference threads=1 so atomic-mode IB is ordered):
  cavity10.npz   C1-style cavity 10^3, 30 steps: f, rho, u
  sphere_ib.npz  sphere IB 24x16x16, 20 steps: rho, u, totals, samples
  fins_ib.npz    rotating fin comb 40x24x24, 20 steps: samples, totals
  c1_anchor.npz  C1 64^3 (SURVEY §8(c) recommended), scalars at t=100 and t=1000
  kats.npz       SPEC.md examples (morton3, split_domain, feq(1,0), ...)
  c2_anchor.npz  C2 256x128x128 sphere + IB: mass, max|u|,
                 reaction force at t=100/200/300 and the z=64 rho/u planes at
                 t=300 (reference on all host threads: atomic-mode spreading,
                 so the last digits vary at ~1e-15 relative)

    python tests/golden/make_golden.py c2     # only c2_anchor.npz (~5 min)
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

import paper_2101_11856_b200 as lbm  # noqa: E402
from oracle import refpy  # noqa: E402
from tests import scenes  # noqa: E402
from tests.test_oracle import _small_fins  # noqa: E402


def _run(cfg, steps, samples=None):
    r = refpy.RefRunner(cfg, threads=1, samples=samples)
    st = r.advance(steps)
    assert st["ok"], st
    return r


def c2_anchor():
    cfg = scenes.sphere()
    r = refpy.RefRunner(cfg)
    out = {}
    for t in (100, 200, 300):
        st = r.advance(t - r.step_count())
        assert st["ok"], st
        rho, u = r.gather_rho(), r.gather_u()
        out[f"mass_{t}"] = rho.sum()
        out[f"umax_{t}"] = np.sqrt((u ** 2).sum(axis=1)).max()
        out[f"force_{t}"] = r.totals_log()[-1][:3]
    out["rho_plane_300"] = rho.reshape(128, 128, 256)[64]
    out["u_plane_300"] = u.reshape(128, 128, 256, 3)[64]
    out["samples"] = len(r.samples(0, 0)["source_id"])
    np.savez_compressed(HERE / "c2_anchor.npz", **out)
    print({k: v for k, v in out.items() if np.ndim(v) <= 1})


def main():
    if sys.argv[1:] == ["c2"]:
        c2_anchor()
        return
    cfg = scenes.cavity(n=10)
    r = _run(cfg, 30)
    np.savez_compressed(HERE / "cavity10.npz", f=r.gather_f(), rho=r.gather_rho(), u=r.gather_u(), steps=30)

    cfg = scenes.sphere(24, 16, 16, center=(8, 8, 8), radius=3.0, subdiv=2, r=0.6)
    r = _run(cfg, 20)
    s = r.samples(0, 0)
    sc = r.scene_samples(0)
    np.savez_compressed(HERE / "sphere_ib.npz", rho=r.gather_rho(), u=r.gather_u(),
                        totals=r.totals_log(), steps=20, scene_positions=sc["positions"],
                        scene_reference=sc["reference_positions"], scene_source=sc["source_id"],
                        **{f"s_{k}": v for k, v in s.items()})

    cfg = _small_fins()
    r = _run(cfg, 20)
    s = r.samples(0, 0)
    np.savez_compressed(HERE / "fins_ib.npz", totals=r.totals_log(),
                        steps=20, **{f"s_{k}": v for k, v in s.items()})

    cfg = scenes.cavity(n=64)
    r = refpy.RefRunner(cfg)
    out = {}
    for t in (100, 1000):
        r.advance(t - r.step_count())
        rho, u = r.gather_rho(), r.gather_u()
        out[f"mass_{t}"] = rho.sum()
        out[f"ke_{t}"] = 0.5 * (rho * (u ** 2).sum(axis=1)).sum()
        out[f"umax_{t}"] = np.sqrt((u ** 2).sum(axis=1)).max()
        out[f"rho_slice_{t}"] = rho.reshape(64, 64, 64)[32]
        out[f"u_slice_{t}"] = u.reshape(64, 64, 64, 3)[:, 32]
    np.savez_compressed(HERE / "c1_anchor.npz", **out)

    kats = {
        "morton_in": np.array([[1, 1, 1], [3, 5, 7], [0, 0, 1], [1 << 20, 3, 9]], dtype=np.uint32),
        "morton_out": np.array([refpy.ref_morton3(1, 1, 1), refpy.ref_morton3(3, 5, 7), refpy.ref_morton3(0, 0, 1),
                                refpy.ref_morton3(1 << 20, 3, 9)], dtype=np.uint64),
        "split_8_4": np.array(refpy.ref_split_domain(8, 4)),
        "split_10_4": np.array(refpy.ref_split_domain(10, 4)),
        "split_7_2": np.array(refpy.ref_split_domain(7, 2)),
        "feq_1_0": refpy.ref_equilibrium(1.0, np.zeros(3)),
        "feq_1_u": refpy.ref_equilibrium(1.02, np.array([0.05, -0.02, 0.01])),
    }
    np.savez_compressed(HERE / "kats.npz", **kats)
    c2_anchor()
    for p in sorted(HERE.glob("*.npz")):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()
