"""Smoke tracers (tracer.hpp / tracer.cpp, runner.cpp:213-223): emission is
bit-exact with the reference's mt19937_64 stream (CPU tests); the device
emit -> advect -> retire step matches the unmodified reference Runner
(oracle/_ref) on the same scene: same live count, same birth steps (integer,
exact), positions within POS_TOL after N steps (the advecting velocity is
the fp32 u*, rel-L2 <= 1e-4 against the FP64 reference, integrated over N
steps); rasterize_density matches the reference's to FP64 rounding.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_2101_11856_b200 as lbm
from oracle import refpy
from tests import scenes

POS_TOL = 1e-3      # max |x_gpu - x_ref| (lattice units) after <= 600 steps
DENSITY_TOL = 1e-12  # per cell, FP64 atomics vs the reference's sequential sums

needs_ref = pytest.mark.skipif(not refpy.ref_available(), reason="oracle/_ref not built (make -C oracle ref)")

EMITTERS = [
    lbm.TracerEmitter(lo=(1.0, 2.0, 3.0), hi=(5.5, 6.25, 7.0), rate=17),
    lbm.TracerEmitter(lo=(0.0, 0.0, 0.0), hi=(0.0, 10.0, 10.0), rate=0),
    lbm.TracerEmitter(lo=(-4.0, -1.0, 2.0), hi=(3.0, 9.0, 4.0), rate=5),
]


# ---- CPU: emission, parsing --------------------------------------------------

@needs_ref
@pytest.mark.parametrize("seed", [1, 7, 2**63 + 5])
@pytest.mark.parametrize("step", [0, 1, 2, 999, 123456789])
def test_emission_bit_exact(seed, step):
    got = lbm.emit_tracers(EMITTERS, step, seed)
    want = refpy.ref_emit_tracers(EMITTERS, step, seed)
    assert got.shape == (22, 3)
    assert np.array_equal(got, want)


def test_emission_is_deterministic_per_step():
    a = lbm.emit_tracers(EMITTERS, 5, 3)
    assert np.array_equal(a, lbm.emit_tracers(EMITTERS, 5, 3))
    assert not np.array_equal(a, lbm.emit_tracers(EMITTERS, 6, 3))
    lo, hi = np.array(EMITTERS[0].lo), np.array(EMITTERS[0].hi)
    assert np.all(a[:17] >= lo) and np.all(a[:17] <= hi)


HEAD = """{"grid": {"nx": 8, "ny": 8, "nz": 8}, "viscosity": 0.02,
      "collision": {"kind": "cm-mrt", "high_order_rate": 1.5, "policy": "relax-toward-one"},
      "faces": {"x-": {"condition": "no-slip"}, "x+": {"condition": "no-slip"},
                "y-": {"condition": "no-slip"}, "y+": {"condition": "no-slip"},
                "z-": {"condition": "no-slip"}, "z+": {"condition": "no-slip"}}, """


def test_tracers_json_key_parsed():
    cfg = lbm.parse_scene_config(HEAD + """
        "tracers": [{"region": {"lo": [1, 1, 1], "hi": [2, 3, 4]}, "rate": 3},
                    {"region": {"lo": [0, 0, 0], "hi": [1, 1, 1]}, "rate": 0}]}""")
    assert [e.rate for e in cfg.emitters] == [3, 0]
    assert tuple(cfg.emitters[0].hi) == (2.0, 3.0, 4.0)


@pytest.mark.parametrize("bad,msg", [
    ('[{"region": {"lo": [1, 1, 1], "hi": [2, 3, 4]}, "rate": -1}]', "rate"),
    ('[{"region": {"lo": [1, 1, 1], "hi": [2, 3, 4]}, "rate": 1, "x": 0}]', "x"),
    ('[{"region": {"lo": [1, 1], "hi": [2, 3, 4]}, "rate": 1}]', "lo"),
])
def test_tracers_json_errors(bad, msg):
    with pytest.raises(lbm.ConfigError, match=msg):
        lbm.parse_scene_config(HEAD + '"tracers": %s}' % bad)


def test_scene_rejects_out_of_range_rate():
    cfg = scenes.cavity(n=8)
    cfg.emitters = [lbm.TracerEmitter(lo=(1, 1, 1), hi=(2, 2, 2), rate=2_000_000)]
    with pytest.raises(lbm.ConfigError, match="rate"):
        lbm.build_scene(cfg)


@needs_ref
def test_reference_rasterize_is_partition_of_unity():
    pos = np.random.default_rng(3).uniform(-1.0, 9.0, size=(200, 3))
    vol = refpy.ref_rasterize_density(pos, (8, 7, 6))
    assert abs(vol.sum() - 200) < 1e-9


# ---- GPU: device tracers against the reference Runner ------------------------

def _channel(emitters):
    """Open duct: x- inlet, x+ outflow, walls elsewhere; tracers leave through x+."""
    cfg = scenes.acm(lbm.SceneConfig(nx=32, ny=16, nz=16, viscosity=0.02))
    cfg.faces = scenes.faces("inlet", "outflow", "no-slip", "no-slip", "no-slip", "no-slip")
    cfg.init_velocity = (0.05, 0.0, 0.0)
    cfg.emitters = emitters
    cfg.seed = 11
    return cfg


DUCT_EMITTERS = [
    lbm.TracerEmitter(lo=(0.5, 2.0, 2.0), hi=(4.0, 13.0, 13.0), rate=20),
    # mostly outside the grid: retired on emission (tombstones -> compaction)
    lbm.TracerEmitter(lo=(-6.0, -6.0, 4.0), hi=(6.0, 6.0, 12.0), rate=12),
]


def _assert_clouds_match(g_cloud, ref):
    pos_r, birth_r = ref
    assert g_cloud.size() == len(birth_r)
    assert np.array_equal(g_cloud.birth_step, birth_r)
    assert np.max(np.abs(g_cloud.positions - pos_r), initial=0.0) <= POS_TOL


@pytest.mark.gpu
@pytest.mark.parametrize("chunks", [1, 6])
def test_tracers_match_reference(chunks):
    cfg = _channel(DUCT_EMITTERS)
    g = lbm.Runner(lbm.build_scene(cfg))
    r = refpy.RefRunner(cfg)
    steps = 600
    for _ in range(chunks):
        assert g.advance(steps // chunks).ok
        assert r.advance(steps // chunks)["ok"]
        _assert_clouds_match(g.tracers(), r.tracers())
    cloud = g.tracers()
    # the out-of-grid share of emitter 2 is retired on emission, flow leaves through x+
    assert 0 < cloud.size() < 600 * (20 + 6)
    assert np.all(np.diff(cloud.birth_step) >= 0)  # emission order kept


@pytest.mark.gpu
def test_tracers_region_count_bitwise():
    cfg = _channel(DUCT_EMITTERS)
    a = lbm.Runner(lbm.build_scene(cfg), regions=1)
    b = lbm.Runner(lbm.build_scene(cfg), regions=3)
    for _ in range(4):
        a.advance(50)
        b.advance(50)
    ca, cb = a.tracers(), b.tracers()
    assert np.array_equal(ca.birth_step, cb.birth_step)
    assert np.array_equal(ca.positions, cb.positions)


@pytest.mark.gpu
def test_tracers_clone_and_timings():
    cfg = _channel(DUCT_EMITTERS)
    a = lbm.Runner(lbm.build_scene(cfg))
    a.advance(37)
    b = a.clone()
    a.advance(20)
    b.advance(20)
    assert np.array_equal(a.tracers().positions, b.tracers().positions)
    rows = []
    a.advance(3, timings=rows)
    assert sum(1 for x in rows if x.phase == "tracers") == 3


@pytest.mark.gpu
def test_tracer_density_matches_reference_rasterize():
    cfg = _channel(DUCT_EMITTERS)
    g = lbm.Runner(lbm.build_scene(cfg))
    g.advance(120)
    cloud = g.tracers()
    vol = g.tracer_density()
    want = refpy.ref_rasterize_density(cloud.positions, cfg.dims)
    assert np.max(np.abs(vol - want)) <= DENSITY_TOL
    assert abs(vol.sum() - cloud.size()) < 1e-8
    host = lbm.rasterize_density(cloud, cfg.dims)
    assert np.max(np.abs(host - want)) <= DENSITY_TOL


@pytest.mark.gpu
def test_no_emitters_no_tracers():
    g = lbm.Runner(lbm.build_scene(scenes.cavity(n=12)))
    g.advance(5)
    assert g.tracers().size() == 0
    assert g.tracer_density().sum() == 0.0


@pytest.mark.gpu
def test_tracers_match_reference_regions_and_moving_solid():
    """Tracers over a rotating fin comb (IB forcing in u*), the device run on
    one region, the reference on two (its sampler crosses the seam through
    the exchanged ghost plane)."""
    cfg = scenes.rotating_fins()
    cfg.emitters = [lbm.TracerEmitter(lo=(30.0, 10.0, 10.0), hi=(100.0, 52.0, 52.0), rate=16)]
    g = lbm.Runner(lbm.build_scene(cfg))
    r = refpy.RefRunner(cfg, regions=2)
    assert g.advance(120).ok
    assert r.advance(120)["ok"]
    _assert_clouds_match(g.tracers(), r.tracers())
