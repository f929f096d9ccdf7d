"""Parity at the BASELINE configs' stated sizes: the
sm_100a engine through the C ABI against the unmodified reference
(oracle/_ref, FP64, all host threads) on the same inputs.

  * C2 (configs[1]) at full size, 256x128x128 + 8,329 IB samples, 300 steps:
    rel-L2 of rho*/u* and the reaction force at t = 100/200/300 against the
    live reference, and mass / max|u| / force against the SURVEY §8(c) anchor
    table (tests/golden/c2_anchor.npz, written by the reference itself through
    tests/golden/make_golden.py);
  * C3 (configs[2]) 128^3 twin, 200 steps, on 1, 2 and 4 z-slab regions;
  * C4 (configs[3]) 150x64x105 twin with 12 seeded boxes (Poisson r = 0.7),
    300 steps;
  * C5 (configs[4]) 128x64x64 twin: 8-fin comb rotating about x, 300 steps.

Tolerances (as in test_gpu_parity.py): rel-L2(rho) <= 1e-6, rel-L2(u) <=
1e-4 after N steps; integer outputs (sample order, flags) and the rigid-motion
positions / boundary velocities bit-exact; reaction force within 1e-3 of the
reference's magnitude (fp32 atomics reorder the spreading sums).
"""
import os
import pathlib

import numpy as np
import pytest

import paper_2101_11856_b200 as lbm
from oracle import refpy
from tests import scenes
from tests.test_gpu_parity import RHO_TOL, U_TOL, rel_l2

pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 1
GOLD = pathlib.Path(__file__).parent / "golden"
F_REL = 1e-3


def _umax(u):
    return float(np.sqrt((u ** 2).sum(axis=1)).max())


def _check_samples_exact(g, r, n_solids, moving=False):
    for s in range(n_solids):
        a, b = g.samples(0, s), r.samples(0, s)
        assert np.array_equal(a["source_id"], b["source_id"])
        assert np.array_equal(a["flagged"], b["flagged"])
        assert np.array_equal(a["positions"], b["positions"])
        if moving:
            assert np.array_equal(a["boundary_velocity"], b["boundary_velocity"])


def _check_totals(g, r):
    tg, tr = g.totals_log(), r.totals_log()
    assert tg.shape == tr.shape
    F = np.abs(tr[:, :3]).max()
    assert np.abs(tg[:, :3] - tr[:, :3]).max() <= F_REL * F + 1e-6


def test_c2_full_size_300_steps_matches_reference_and_anchors():
    cfg = scenes.sphere()
    g = lbm.Runner(lbm.build_scene(cfg))
    r = refpy.RefRunner(cfg, threads=THREADS)
    gold = np.load(GOLD / "c2_anchor.npz")
    assert len(g.samples(0, 0)["source_id"]) == int(gold["samples"]) == 8329
    for t in (100, 200, 300):
        sg = g.advance(t - g.step_count())
        sr = r.advance(t - r.step_count())
        assert sg.ok and sr["ok"] and g.step_count() == r.step_count() == t
        rho_g, u_g = g.gather_rho(), g.gather_u()
        rho_r, u_r = r.gather_rho(), r.gather_u()
        assert rel_l2(rho_g, rho_r) <= RHO_TOL, (t, rel_l2(rho_g, rho_r))
        assert rel_l2(u_g, u_r) <= U_TOL, (t, rel_l2(u_g, u_r))
        mass = rho_g.sum()
        for ref_mass in (rho_r.sum(), float(gold[f"mass_{t}"])):
            assert abs(mass - ref_mass) / ref_mass <= 1e-7, (t, mass, ref_mass)
        for ref_umax in (_umax(u_r), float(gold[f"umax_{t}"])):
            assert abs(_umax(u_g) - ref_umax) / ref_umax <= 1e-3, (t, _umax(u_g), ref_umax)
        fg = g.totals_log()[-1][:3]
        for ref_f in (r.totals_log()[-1][:3], gold[f"force_{t}"]):
            assert np.abs(fg - ref_f).max() <= F_REL * np.abs(ref_f).max() + 1e-6, (t, fg, ref_f)
    assert rel_l2(g.gather_rho().reshape(128, 128, 256)[64], gold["rho_plane_300"]) <= RHO_TOL
    assert rel_l2(g.gather_u().reshape(128, 128, 256, 3)[64], gold["u_plane_300"]) <= U_TOL
    _check_totals(g, r)
    _check_samples_exact(g, r, 1)


@pytest.fixture(scope="module")
def c3_twin_reference():
    cfg = scenes.channel(n=128)
    r = refpy.RefRunner(cfg, threads=THREADS)
    st = r.advance(200)
    assert st["ok"]
    return cfg, r.gather_rho(), r.gather_u()


@pytest.mark.parametrize("regions", [1, 2, 4])
def test_c3_twin_128_cubed(c3_twin_reference, regions):
    cfg, rho_r, u_r = c3_twin_reference
    g = lbm.Runner(lbm.build_scene(cfg), regions=regions)
    st = g.advance(200)
    assert st.ok and g.step_count() == 200
    assert rel_l2(g.gather_rho(), rho_r) <= RHO_TOL
    assert rel_l2(g.gather_u(), u_r) <= U_TOL, rel_l2(g.gather_u(), u_r)


def test_c4_city_twin_300_steps():
    cfg = scenes.city_twin()
    g = lbm.Runner(lbm.build_scene(cfg))
    r = refpy.RefRunner(cfg, threads=THREADS)
    for t in (100, 200, 300):
        sg = g.advance(t - g.step_count())
        sr = r.advance(t - r.step_count())
        assert sg.ok and sr["ok"]
        assert rel_l2(g.gather_rho(), r.gather_rho()) <= RHO_TOL
        assert rel_l2(g.gather_u(), r.gather_u()) <= U_TOL, (t, rel_l2(g.gather_u(), r.gather_u()))
    _check_totals(g, r)
    _check_samples_exact(g, r, len(cfg.solids))


def test_c5_rotating_fan_twin_300_steps():
    cfg = scenes.rotating_fins()  # 128x64x64, 8 fins, omega = 2 pi / 500 about x
    g = lbm.Runner(lbm.build_scene(cfg))
    r = refpy.RefRunner(cfg, threads=THREADS)
    for t in (100, 200, 300):
        sg = g.advance(t - g.step_count())
        sr = r.advance(t - r.step_count())
        assert sg.ok and sr["ok"]
        assert rel_l2(g.gather_rho(), r.gather_rho()) <= RHO_TOL
        assert rel_l2(g.gather_u(), r.gather_u()) <= U_TOL, (t, rel_l2(g.gather_u(), r.gather_u()))
        _check_samples_exact(g, r, 1, moving=True)
    _check_totals(g, r)
    a, b = g.samples(0, 0), r.samples(0, 0)
    pf = np.abs(b["penalty_force"]).max()
    assert np.abs(a["penalty_force"] - b["penalty_force"]).max() <= F_REL * pf + 1e-9
