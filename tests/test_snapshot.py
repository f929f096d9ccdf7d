"""Snapshot / readback path: LBF1 field dumps byte-identical
to the reference's dump_field and readable by its load_field; the
asynchronous device snapshot equals the synchronous gather of the same step."""
import numpy as np
import pytest

import paper_2101_11856_b200 as lbm
from oracle import refpy
from tests import scenes


def test_dump_field_bytes_match_reference(tmp_path):
    rng = np.random.default_rng(3)
    dims = (5, 4, 3)
    for beta in (1, 3, 27):
        a = rng.standard_normal(60 * beta)
        ours, ref = tmp_path / f"o{beta}.lbf", tmp_path / f"r{beta}.lbf"
        lbm.dump_field(ours, dims, a)
        refpy.ref_dump_field(ref, dims, a)
        assert ours.read_bytes() == ref.read_bytes()
        d, b, back = refpy.ref_load_field(ours, a.size)
        assert d == dims and b == beta and np.array_equal(back, a)


def test_dump_field_rejects_bad_size(tmp_path):
    with pytest.raises(lbm.ConfigError):
        lbm.dump_field(tmp_path / "x.lbf", (2, 2, 2), np.zeros(7))


@pytest.mark.gpu
@pytest.mark.parametrize("make", [lambda: scenes.cavity(n=24),
                                  lambda: scenes.sphere(48, 32, 32, center=(16, 16, 16), radius=5.0, subdiv=3,
                                                        r=0.6)])
def test_async_snapshot_matches_gather_while_stepping(make, tmp_path):
    cfg = make()
    g = lbm.Runner(lbm.build_scene(cfg))
    g.advance(20)
    rho20, u20 = g.gather_rho(), g.gather_u()
    g.snapshot_begin()
    g.advance(7)           # the step loop continues while the snapshot drains
    g.advance(5)
    t, rho, u = g.snapshot_wait()
    assert t == 20
    assert np.array_equal(rho, rho20) and np.array_equal(u, u20.reshape(-1, 3))
    assert g.step_count() == 32
    # the runner's own state is unaffected by the snapshot
    ref = lbm.Runner(lbm.build_scene(cfg))
    ref.advance(20)
    ref.advance(12)
    assert np.allclose(g.gather_f(), ref.gather_f(), rtol=0, atol=1e-5)
    path = tmp_path / "rho.lbf"
    lbm.dump_field(path, (cfg.nx, cfg.ny, cfg.nz), rho)
    d, b, back = refpy.ref_load_field(path, rho.size)
    assert b == 1 and np.array_equal(back, rho)
