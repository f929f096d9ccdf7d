"""The step's execution variants against each other (GPU).

Each variant is a process-wide switch read once, so every run is a child
process: the per-step ghost fill replayed from its resolved copy program
(default) vs the general per-entry kernel (LBMG_FILL_PLAN=0); rho*/u*
recomputed on demand from f(t) of the last step (default) vs stored by the
last step's fluid kernel (LBMG_LAZY_MACRO=0); the fill program as extra blocks
of the IB launch (default) vs a fill || IB fork/join (LBMG_IB_MERGE=0).  The
first two are exact rewrites of the same arithmetic: bitwise.  The merged
launch only changes when the IB's fp32 REDs land: within the IB tolerance of
test_gpu_parity.py."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]

CHILD = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np
import paper_2101_11856_b200 as lbm
from tests import scenes
cfg = getattr(scenes, {scene!r})(**{kw!r})
r = lbm.Runner(lbm.build_scene(cfg))
if {variant!r} is not None:
    r.set_variant(*{variant!r})
for n in {chunks!r}:
    st = r.advance(n)
out = dict(rho=r.gather_rho(), u=r.gather_u(), f=r.gather_f(), t=np.array([r.step_count()]))
if cfg.solids:
    out["force"] = r.samples(0, 0)["penalty_force"]
    out["totals"] = r.totals_log()
np.savez({out!r}, **out)
"""


def _run(tmp_path, tag, env_extra, scene, kw, chunks, variant=None):
    out = tmp_path / f"{tag}.npz"
    env = dict(os.environ, **env_extra)
    code = CHILD.format(root=str(ROOT), scene=scene, kw=kw, chunks=chunks, out=str(out), variant=variant)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return dict(np.load(out))


def _bitwise(a, b):
    assert a.keys() == b.keys()
    for k in a:
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.gpu
@pytest.mark.parametrize("scene,kw", [
    ("outflow_mix", dict(nx=24, ny=20, nz=16)),  # inlet, outflow edges (stale face-slot reads), no-slip
    ("channel", dict(n=32)),                       # x/z periodic wraps, y walls, one periodic region
])
def test_fill_program_and_lazy_macro_are_bitwise(tmp_path, scene, kw):
    chunks = [7, 1, 12]
    base = _run(tmp_path, "base", {}, scene, kw, chunks)
    _bitwise(base, _run(tmp_path, "noplan", {"LBMG_FILL_PLAN": "0"}, scene, kw, chunks))
    _bitwise(base, _run(tmp_path, "eager", {"LBMG_LAZY_MACRO": "0"}, scene, kw, chunks))


@pytest.mark.gpu
def test_merged_ib_fill_launch_matches_fork_join(tmp_path):
    kw = dict(nx=64, ny=40, nz=40, center=(24, 20, 20), radius=6.0, subdiv=3, r=0.6)
    chunks = [10, 1, 9]
    a = _run(tmp_path, "merged", {}, "sphere", kw, chunks)
    b = _run(tmp_path, "fork", {"LBMG_IB_MERGE": "0"}, "sphere", kw, chunks)
    c = _run(tmp_path, "eager", {"LBMG_LAZY_MACRO": "0", "LBMG_FILL_PLAN": "0"}, "sphere", kw, chunks)
    for other in (b, c):
        assert int(a["t"][0]) == int(other["t"][0]) == sum(chunks)
        assert np.abs(a["f"] - other["f"]).max() <= 2e-5
        for k in ("rho", "u", "force", "totals"):
            rel = np.linalg.norm(a[k] - other[k]) / max(np.linalg.norm(other[k]), 1e-30)
            assert rel <= 1e-4, (k, rel)


@pytest.mark.gpu
@pytest.mark.parametrize("scene,kw", [
    ("city", dict(nx=64, ny=32, nz=48, n_boxes=4)),   # static boxes on the ground (supports on ghost slots)
    ("sphere", dict(nx=64, ny=40, nz=40, center=(24, 20, 20), radius=6.0, subdiv=3, r=0.6)),
])
def test_ib_band_path_matches_gathers(tmp_path, scene, kw):
    """The fused IB kernel reading per-corner moments from the band list
    (LBMG_IB_BAND=1; default above 64 k static samples) vs gathering the 27
    populations per corner: the same sums in the same order, so only the fp32
    RED arrival order differs."""
    chunks = [10, 1, 9]
    a = _run(tmp_path, "band", {"LBMG_IB_BAND": "1"}, scene, kw, chunks)
    b = _run(tmp_path, "gather", {"LBMG_IB_BAND": "0"}, scene, kw, chunks)
    assert int(a["t"][0]) == int(b["t"][0]) == sum(chunks)
    assert np.abs(a["f"] - b["f"]).max() <= 2e-5
    for k in ("rho", "u", "force", "totals"):
        rel = np.linalg.norm(a[k] - b[k]) / max(np.linalg.norm(b[k]), 1e-30)
        assert rel <= 1e-4, (k, rel)


@pytest.mark.gpu
def test_split_pipeline_shared_memory_scatter_matches_direct(tmp_path):
    """The split IB pipeline's spread with per-CTA shared-memory pre-aggregation
    (LBMG_IB_SPREAD=smem: one global RED per distinct node and component) vs
    one RED per corner, and both vs the fused kernel."""
    kw = dict(nx=64, ny=40, nz=40, center=(24, 20, 20), radius=6.0, subdiv=3, r=0.6)
    chunks = [10, 1, 9]
    a = _run(tmp_path, "smem", {"LBMG_IB_SPREAD": "smem"}, "sphere", kw, chunks, variant=(0, 1))
    b = _run(tmp_path, "direct", {}, "sphere", kw, chunks, variant=(0, 1))
    c = _run(tmp_path, "fused", {}, "sphere", kw, chunks)
    for other in (b, c):
        assert int(a["t"][0]) == int(other["t"][0]) == sum(chunks)
        assert np.abs(a["f"] - other["f"]).max() <= 2e-5
        for k in ("rho", "u", "force", "totals"):
            rel = np.linalg.norm(a[k] - other[k]) / max(np.linalg.norm(other[k]), 1e-30)
            assert rel <= 1e-4, (k, rel)
