"""Eq. 10 auto-tuner (SPEC [MODULE] autotune; autotune.cpp): candidate grid,
argmin + tie rule against the unmodified reference's search_with_cost on
injected cost tables, and (GPU) a real device sweep that never alters physics."""
import math

import numpy as np
import pytest

import paper_2101_11856_b200 as lbm
from paper_2101_11856_b200 import autotune
from oracle import refpy
from tests import scenes


def test_spec_example_fake_cost_minimum():
    # SPEC autotune example: known minimum at (ell=2, alpha=2^6) -> (2, 64)
    spec = autotune.TuneSpec(ell_min=1, ell_max=4, alphas=[2 ** k for k in range(1, 11)])
    out = autotune.search_with_cost(spec, lambda l, a: abs(l - 2) + abs(math.log2(a) - 6) + 1.0)
    assert (out.ell, out.alpha) == (2, 64)
    assert len(out.rows) == spec.candidate_count() == 40


def test_single_candidate_and_all_invalid():
    spec = autotune.TuneSpec(ell_min=3, ell_max=3, alphas=[8])
    out = autotune.search_with_cost(spec, lambda l, a: 0.5)
    assert (out.ell, out.alpha, out.cost) == (3, 8, 0.5)
    with pytest.raises(lbm.ConfigError):
        autotune.search_with_cost(spec, lambda l, a: math.inf)


@pytest.mark.parametrize("seed", range(6))
def test_argmin_and_ties_match_reference(seed):
    rng = np.random.default_rng(seed)
    ell_min, ell_max = 1, 5
    alphas = [2 ** k for k in range(1, 9)]
    # coarse values -> many ties; some invalid candidates
    table = rng.integers(1, 4, size=(ell_max - ell_min + 1, len(alphas))).astype(float)
    table[rng.random(table.shape) < 0.2] = math.inf
    spec = autotune.TuneSpec(ell_min=ell_min, ell_max=ell_max, alphas=alphas)
    ours = autotune.search_with_cost(spec, lambda l, a: table[l - ell_min, alphas.index(a)])
    ref = refpy.ref_search_with_cost(ell_min, ell_max, alphas, table.ravel())
    assert (ours.ell, ours.alpha, ours.cost) == ref


def test_variant_dimension_is_outermost_with_ties_to_default():
    spec = autotune.TuneSpec(ell_min=1, ell_max=2, alphas=[2, 4], variants=[(0, 0), (1, 0)])
    out = autotune.search_with_cost(spec, lambda l, a, v: 1.0)
    assert (out.variant, out.ell, out.alpha) == ((0, 0), 1, 2)
    out = autotune.search_with_cost(spec, lambda l, a, v: 1.0 if v == (1, 0) and (l, a) == (2, 4) else 2.0)
    assert (out.variant, out.ell, out.alpha) == ((1, 0), 2, 4)


def test_tune_spec_ranges_match_reference():
    cfg = scenes.sphere(48, 32, 32, center=(16, 16, 16), radius=5.0, subdiv=3, r=0.6)
    scene = lbm.build_scene(cfg)
    ours = autotune.TuneSpec.from_scene(scene, n_steps=10, warmup=5)
    r = refpy.RefRunner(cfg)
    lo, hi, alphas = refpy.ref_tune_spec(r, 10, 5)
    assert (ours.ell_min, ours.ell_max, ours.alphas) == (lo, hi, alphas)


@pytest.mark.gpu
def test_device_search_never_alters_physics():
    cfg = scenes.sphere(48, 32, 32, center=(16, 16, 16), radius=5.0, subdiv=3, r=0.6)
    scene = lbm.build_scene(cfg)
    base = lbm.Runner(scene)
    base.advance(5)
    f0 = base.gather_f()
    spec = autotune.TuneSpec.from_scene(scene, n_steps=3, warmup=1,
                                        variants=[(0, 0), (0, 1), (1, 1)])
    spec.ell_max = min(spec.ell_max, 3)
    spec.alphas = [a for a in spec.alphas if a in (2, 64, 256, 4096, 1 << 15)]
    out = autotune.search(base, spec)
    assert len(out.rows) == spec.candidate_count()
    assert math.isfinite(out.cost) and out.cost > 0
    assert all(r.seconds > 0 for r in out.rows)
    assert base.step_count() == 5 and np.array_equal(base.gather_f(), f0)  # search ran on a clone
    # the tuned configuration reproduces the default run (layout/variant invariance)
    ref = lbm.Runner(scene)
    ref.advance(12)
    tuned = lbm.Runner(scene)
    autotune.apply(tuned, out)
    tuned.advance(12)
    assert np.abs(tuned.gather_f() - ref.gather_f()).max() <= 2e-5  # fp32 IB atomics order only


def test_cta_shape_dimension_in_search():
    """Variants may carry the staged kernel's CTA shape as a third entry."""
    spec = autotune.TuneSpec(ell_min=1, ell_max=1, alphas=[2, 4],
                             variants=[(0, 0, 512), (0, 0, 256), (0, 0, 128)])
    assert spec.candidate_count() == 6
    out = autotune.search_with_cost(spec, lambda l, a, v: {512: 3.0, 256: 2.0, 128: 2.0}[v[2]])
    assert out.variant == (0, 0, 256) and out.alpha == 2  # ties keep the earlier candidate


@pytest.mark.gpu
def test_cta_shapes_are_bitwise_identical_and_searchable():
    cfg = scenes.channel(n=32, nz=40)
    scene = lbm.build_scene(cfg)
    outs = []
    for cta in (512, 256, 128):
        r = lbm.Runner(scene)
        r.set_cta(cta)
        assert r.cta() == cta
        r.advance(7)
        outs.append(r.gather_f())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    with pytest.raises(lbm.ConfigError):
        lbm.Runner(scene).set_cta(96)
    base = lbm.Runner(scene)
    spec = autotune.TuneSpec(ell_min=1, ell_max=1, alphas=[1 << 20], n_steps=2, warmup=1,
                             variants=[(0, 0, 512), (0, 0, 256), (0, 0, 128)])
    out = autotune.search(base, spec)
    assert len(out.rows) == 3 and all(math.isfinite(r.seconds) for r in out.rows)
    tuned = lbm.Runner(scene)
    autotune.apply(tuned, out)
    assert tuned.cta() == out.variant[2]
