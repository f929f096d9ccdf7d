"""Pin the plain-C restatement oracle (oracle/lbm_oracle.c) against the
unmodified reference (oracle/_ref): bit-identical FP64 on every step
function, integer helper and whole-run field, plus the SPEC examples."""
import numpy as np
from pathlib import Path
import pytest

import paper_2101_11856_b200 as lbm
from oracle import refpy
from tests import scenes


def _samples(cfg):
    if not cfg.solids:
        return []
    sc = lbm.build_scene(cfg)
    return [sc.samples(s) for s in range(len(cfg.solids))]


def test_lattice_and_rows():
    import ctypes as C
    c = (C.c_int * 81)()
    w = np.zeros(27)
    opp = (C.c_int * 27)()
    q = (C.c_int * 81)()
    refpy.oracle_lib().orc_lattice(c, refpy._dp(w), opp, q)
    rc, rw, ropp = refpy.ref_lattice()
    rq, _ = refpy.ref_moment_exponents()
    assert np.array_equal(np.array(c[:]).reshape(27, 3), rc)
    assert np.array_equal(w, rw)
    assert np.array_equal(np.array(opp[:]), ropp)
    assert np.array_equal(np.array(q[:]).reshape(27, 3), rq)


@pytest.mark.parametrize("kind,policy,hor", [("bgk", "constant", 1.0), ("rm-mrt", "constant", 1.3),
                                             ("rm-mrt", "relax-toward-one", 1.3),
                                             ("cm-mrt", "constant", 1.5), ("cm-mrt", "relax-toward-one", 1.5)])
def test_collide_bitwise(kind, policy, hor):
    cfg = lbm.SceneConfig(nx=2, ny=2, nz=2, viscosity=0.02, kind=kind, policy=policy, high_order_rate=hor)
    rng = np.random.default_rng(5)
    n = 500
    rho = 1.0 + rng.uniform(-0.05, 0.05, n)
    u = rng.uniform(-0.05, 0.05, (n, 3))
    f = np.stack([refpy.ref_equilibrium(rho[k], u[k]) for k in range(n)]) * (1 + rng.uniform(-0.05, 0.05, (n, 27)))
    assert np.array_equal(refpy.oracle_collide(cfg, f, rho, u), refpy.ref_collide(cfg, f, rho, u))


def test_spec_collision_equivalences():
    """SPEC criterion 4: equal-rate MRT == BGK; conservation of the collision."""
    rng = np.random.default_rng(11)
    n = 300
    rho = 1.0 + rng.uniform(-0.05, 0.05, n)
    u = rng.uniform(-0.05, 0.05, (n, 3))
    f = np.stack([refpy.ref_equilibrium(rho[k], u[k]) for k in range(n)]) * (1 + rng.uniform(-0.05, 0.05, (n, 27)))
    bgk = lbm.SceneConfig(nx=2, ny=2, nz=2, viscosity=0.02, kind="bgk")
    om = 1.0 / (3 * 0.02 + 0.5)
    eq = lbm.SceneConfig(nx=2, ny=2, nz=2, viscosity=0.02, kind="cm-mrt", explicit_rates=[om] * 27)
    assert np.abs(refpy.oracle_collide(bgk, f, rho, u) - refpy.oracle_collide(eq, f, rho, u)).max() <= 1e-13
    c, _, _ = refpy.ref_lattice()
    cm = scenes.acm(lbm.SceneConfig(nx=2, ny=2, nz=2, viscosity=0.02))
    rho_f = f.sum(axis=1)  # consistent moments: the collision conserves them
    u_f = (f @ c) / rho_f[:, None]
    Om = refpy.oracle_collide(cm, f, rho_f, u_f)
    assert np.abs(Om.sum(axis=1)).max() <= 1e-15
    assert np.abs(Om @ c).max() <= 1e-15


def test_equilibrium_spec_example():
    # SPEC.md:159 feq(1, 0) = w exactly
    feq = np.zeros(27)
    u = np.zeros(3)
    refpy.oracle_lib().orc_equilibrium(1.0, refpy._dp(u), refpy._dp(feq))
    _, w, _ = refpy.ref_lattice()
    assert np.array_equal(feq, w)


def test_integer_helpers_bitwise():
    assert refpy.oracle_lib().orc_morton3(1, 1, 1) == 7
    rng = np.random.default_rng(2)
    for x, y, z in rng.integers(0, 1 << 21, size=(100, 3)):
        assert refpy.oracle_lib().orc_morton3(int(x), int(y), int(z)) == refpy.ref_morton3(int(x), int(y), int(z))
    pos = rng.uniform(0, 20, size=(500, 3))
    src = rng.permutation(500).astype(np.uint32)
    for ell in (1, 2, 5):
        assert np.array_equal(refpy.oracle_reorder_permutation(pos, src, ell),
                              refpy.ref_reorder_permutation(pos, src, ell))
    for nz, m in [(8, 4), (10, 4), (7, 2), (33, 5)]:
        assert refpy.oracle_split_domain(nz, m) == refpy.ref_split_domain(nz, m)
    for fs in [("no-slip",) * 6, ("inlet", "outflow", "periodic", "periodic", "outflow", "no-slip")]:
        cfg = scenes.acm(lbm.SceneConfig(nx=5, ny=6, nz=4, viscosity=0.05))
        cfg.faces = scenes.faces(*fs)
        assert np.array_equal(refpy.oracle_face_owner(cfg), refpy.ref_face_owner(cfg))


def _run_both(cfg, steps, chunks=1):
    samples = _samples(cfg)
    o = refpy.OracleRunner(cfg, samples)
    r = refpy.RefRunner(cfg, threads=1, samples=samples if samples else None)
    for _ in range(chunks):
        so = o.advance(steps // chunks)
        sr = r.advance(steps // chunks)
    return o, r, so, sr


CASES = {
    "cavity": (lambda: scenes.cavity(n=10), 30),
    "taylor_green": (lambda: scenes.taylor_green(nx=12, ny=10, nz=4), 30),
    "outflow_mix": (lambda: scenes.outflow_mix(), 25),
    "channel_body_force": (lambda: scenes.channel(n=8, nz=10), 30),
    "sphere_ib": (lambda: scenes.sphere(24, 16, 16, center=(8, 8, 8), radius=3.0, subdiv=2, r=0.6), 20),
    "moving_fins": (lambda: _small_fins(), 20),
    "sphere_ib_det": (lambda: _det(scenes.sphere(24, 16, 16, center=(8, 8, 8), radius=3.0, subdiv=2, r=0.6)), 15),
    "bgk_tg": (lambda: scenes.taylor_green(nx=8, ny=8, nz=4, kind="bgk"), 20),
}


def _det(cfg):
    cfg.ib_mode = "deterministic"
    return cfg


def _small_fins():
    cfg = scenes.rotating_fins(40, 24, 24)
    cfg.solids[0].mesh.origin = (14, 8, 8)
    cfg.solids[0].mesh.fin_length = 8
    cfg.solids[0].mesh.fin_height = 6
    cfg.solids[0].mesh.fins = 3
    cfg.solids[0].motion.center = (18, 10.5, 11)
    cfg.solids[0].motion.angular_velocity = (0.05, 0.0, 0.0)
    return cfg


@pytest.mark.parametrize("name", sorted(CASES))
def test_runner_bitwise_vs_reference(name):
    make, steps = CASES[name]
    cfg = make()
    o, r, so, sr = _run_both(cfg, steps, chunks=2)
    assert so == sr
    assert o.step_count() == r.step_count()
    assert np.array_equal(o.gather_f(), r.gather_f())
    assert np.array_equal(o.gather_rho(), r.gather_rho())
    assert np.array_equal(o.gather_u(), r.gather_u())
    assert np.array_equal(o.totals_log(), r.totals_log())
    for s in range(len(cfg.solids)):
        a, b = o.samples(s), r.samples(0, s)
        for k in ("positions", "boundary_velocity", "penalty_force", "sampled_velocity", "flagged"):
            assert np.array_equal(a[k], b[k]), k


def test_divergence_bitwise():
    cfg = lbm.SceneConfig(nx=8, ny=8, nz=8, viscosity=1e-5, kind="bgk")
    cfg.faces = scenes.faces("inlet", "outflow", "no-slip", "no-slip", "no-slip", "no-slip", inlet=(0.6, 0, 0))
    cfg.init_velocity = (0.6, 0.0, 0.0)
    o, r, so, sr = _run_both(cfg, 2000)
    assert not so["ok"] and so == sr
    assert np.array_equal(o.gather_rho(), r.gather_rho())


def test_c2_anchor_fixture_matches_survey_table():
    # tests/golden/c2_anchor.npz is written by the unmodified reference
    # (make_golden.py c2); SURVEY.md §8(c) recorded the same anchors from an
    # independent probe of the reference: mass, max|u|, reaction force.
    gold = np.load(Path(__file__).parent / "golden" / "c2_anchor.npz")
    table = {100: (4195873.0964478, 0.06738708, (24.07249, 0.1624865, 0.1420280)),
             200: (4197716.8690329, 0.06545837, (13.03389, 0.1435446, 0.1404260)),
             300: (4202373.2614346, 0.06606140, (0.8222260, -0.06475448, -0.04553023))}
    for t, (mass, umax, force) in table.items():
        assert abs(float(gold[f"mass_{t}"]) - mass) <= 1e-7 * mass
        assert abs(float(gold[f"umax_{t}"]) - umax) <= 1e-8
        assert np.allclose(gold[f"force_{t}"], force, rtol=2e-6, atol=1e-9)
    assert int(gold["samples"]) == 8329
