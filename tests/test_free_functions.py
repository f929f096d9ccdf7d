"""The reference's free-function surface on the device:
step() on an explicit single-region state (solver.hpp:82-83) and the IB free
functions (ib.hpp:77-128), each against the unmodified reference's own
function (oracle/_ref) on the same inputs.

Tolerances: kernel support, interpolation, penalty forces and rigid motion
are FP64 with the reference's operation order: bit-exact.  Spreading sums
with FP64 atomics (the reference's atomic mode): 1e-14 relative.  Reaction
totals (fixed-order tree vs the reference's serial sum): 1e-12 relative.
step(): fp32 storage, rel-L2(rho) <= 1e-6, rel-L2(u) <= 1e-4, max|df| <= 2e-6.
"""
import math

import numpy as np
import pytest

import paper_2101_11856_b200 as lbm
from oracle import refpy
from tests import scenes
from tests.test_gpu_parity import F_TOL, RHO_TOL, U_TOL, rel_l2

pytestmark = pytest.mark.gpu


def _state(cfg, seed=3):
    """A non-equilibrium state: feq of a smooth field times (1 + 2% noise)."""
    rng = np.random.default_rng(seed)
    n = cfg.nx * cfg.ny * cfg.nz
    z, y, x = np.meshgrid(np.arange(cfg.nz), np.arange(cfg.ny), np.arange(cfg.nx), indexing="ij")
    rho = 1.0 + 0.01 * np.sin(2 * np.pi * x / cfg.nx).ravel()
    u = np.stack([0.02 * np.cos(2 * np.pi * y / cfg.ny), 0.01 * np.sin(2 * np.pi * z / cfg.nz),
                  0.005 * np.cos(2 * np.pi * x / cfg.nx)], axis=-1).reshape(n, 3)
    f = np.stack([refpy.ref_equilibrium(rho[k], u[k]) for k in range(n)])
    return f * (1 + 0.02 * rng.uniform(-1, 1, f.shape))


@pytest.mark.parametrize("make", [lambda: scenes.outflow_mix(12, 8, 10), lambda: scenes.cavity(n=12),
                                  lambda: scenes.channel(n=12, nz=10)])
def test_step_on_explicit_state_matches_reference(make):
    cfg = make()
    f = _state(cfg)
    f_star = _state(cfg, seed=5)  # the face-pass scratch: its stale face entries matter for outflow edges
    g = lbm.Runner(lbm.build_scene(cfg))
    g.load_state(f, f_star, t=7)
    assert g.step_count() == 7
    for _ in range(3):
        st = g.step()
        assert st.ok
    assert g.step_count() == 10
    fr, rr, ur, sr = refpy.ref_step(cfg, f, f_star, 7, 3)
    assert sr["ok"]
    assert np.abs(g.gather_f() - fr).max() <= F_TOL
    assert rel_l2(g.gather_rho(), rr) <= RHO_TOL
    assert rel_l2(g.gather_u(), ur) <= U_TOL


def test_step_rejects_runners_with_solids():
    cfg = scenes.sphere(32, 20, 20, center=(10, 10, 10), radius=3.0, subdiv=2, r=0.6)
    g = lbm.Runner(lbm.build_scene(cfg))
    with pytest.raises(lbm.StateError):
        g.step()
    with pytest.raises(lbm.StateError):
        g.load_state(np.zeros((32 * 20 * 20, 27)))


def _samples(dims, n=600, seed=9, margin=-0.6):
    rng = np.random.default_rng(seed)
    lo = np.full(3, margin)
    hi = np.array(dims, dtype=float) - 1 - margin
    return rng.uniform(lo, hi, (n, 3))  # some outside the grid (flagged)


def test_ib_free_functions_match_reference():
    dims = (14, 11, 9)
    nodes = dims[0] * dims[1] * dims[2]
    rng = np.random.default_rng(4)
    pos = _samples(dims)
    u = rng.uniform(-0.05, 0.05, (nodes, 3))
    rho = 1.0 + rng.uniform(-0.02, 0.02, nodes)
    ub = rng.uniform(-0.03, 0.03, (len(pos), 3))
    # kernel support, per sample
    base, w, inside = lbm.ib_kernel_support(pos, dims)
    for k in range(0, len(pos), 37):
        ins, b, ww = refpy.ref_kernel_support(pos[k], dims)
        assert ins == inside[k] and tuple(base[k]) == b and np.array_equal(w[k], ww)
    # interpolate -> penalty -> spread, bit-exact where the order is fixed
    us, fl = lbm.ib_interpolate_velocity(pos, u, dims)
    us_r, fl_r = refpy.ref_ib_interpolate_velocity(pos, u, dims)
    assert np.array_equal(fl, fl_r) and fl.any() and not fl.all()
    assert np.array_equal(us, us_r)
    fo = lbm.ib_penalty_forces(pos, ub, us, fl, rho, dims)
    fo_r = refpy.ref_ib_penalty_forces(pos, ub, us_r, fl_r, rho, dims)
    assert np.array_equal(fo, fo_r)
    g0 = rng.uniform(-1e-3, 1e-3, (nodes, 3))
    g = lbm.ib_spread_forces(pos, fo, fl, g0, dims)
    g_r = refpy.ref_ib_spread_forces(pos, fo_r, fl_r, g0, dims)
    assert np.abs(g - g_r).max() <= 1e-14 * np.abs(g_r).max()
    # reaction totals over a slab and the whole grid
    c = np.array([6.5, 5.0, 4.0])
    for z0, z1 in ((0, dims[2]), (2, 6)):
        F, T = lbm.ib_reaction_totals(pos, fo, c, z0, z1)
        F_r, T_r = refpy.ref_ib_reaction_totals(pos, fo_r, c, z0, z1)
        assert np.abs(F - F_r).max() <= 1e-12 * max(np.abs(F_r).max(), 1e-300)
        assert np.abs(T - T_r).max() <= 1e-12 * max(np.abs(T_r).max(), 1e-300)


def test_ib_slab_seam_rule_partitions_the_spread():
    # sample_active + owned-plane spreading (ib.cpp:313-317, :377): the slabs
    # of split_domain spread exactly the whole-grid forces between them
    dims = (12, 10, 16)
    nodes = dims[0] * dims[1] * dims[2]
    rng = np.random.default_rng(8)
    pos = _samples(dims, margin=0.1)
    fo = rng.uniform(-0.01, 0.01, pos.shape)
    fl = np.zeros(len(pos), dtype=np.uint8)
    whole = lbm.ib_spread_forces(pos, fo, fl, np.zeros((nodes, 3)), dims)
    parts = np.zeros((nodes, 3))
    for z0, z1 in lbm.split_domain(dims[2], 3):
        parts += lbm.ib_spread_forces(pos, fo, fl, np.zeros((nodes, 3)), dims, slab=(z0, z1))
    assert np.abs(parts - whole).max() <= 1e-15


def test_ib_rigid_motion_bit_exact():
    dims = (40, 30, 30)
    rng = np.random.default_rng(2)
    ref = rng.uniform(-8, 8, (500, 3))
    motion = lbm.RigidMotion(linear_velocity=(0.01, -0.002, 0.0), angular_velocity=(2 * math.pi / 500, 0.003, -0.001),
                             center=(20.0, 15.0, 15.0))
    for t in (0, 1, 37, 499, 12345):
        a = lbm.ib_update_rigid_motion(ref, motion, t, dims)
        b = refpy.ref_ib_update_rigid_motion(ref, motion, t, dims)
        for x, y in zip(a, b):
            assert np.array_equal(x, y), t
