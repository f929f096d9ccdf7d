"""The C++ drop-in header (include/lbm_b200.hpp) compiles and links like a
reference client; on a GPU box the example runs and matches the Python path."""
import os
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _build(tmp_path):
    exe = tmp_path / "cavity"
    lib = ROOT / "paper_2101_11856_b200" / "_build"
    subprocess.run(["g++", "-std=c++17", "-Wall", "-Werror", f"-I{ROOT / 'include'}", str(ROOT / "examples" / "cavity.cpp"),
                    f"-L{lib}", "-llbmg", f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    return exe


def test_cpp_example_compiles(tmp_path):
    assert _build(tmp_path).exists()


@pytest.mark.gpu
def test_cpp_example_runs(tmp_path):
    exe = _build(tmp_path)
    res = subprocess.run([str(exe), "20"], capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    out = res.stdout
    assert "steps=20 ok=1" in out
    import numpy as np
    import paper_2101_11856_b200 as lbm
    from tests import scenes
    r = lbm.Runner(lbm.build_scene(scenes.cavity(n=64)))
    r.advance(20)
    mass = float(out.split("mass=")[1].split()[0])
    n_tr = int(out.split("tracers=")[1].split()[0])
    assert n_tr == 200 and abs(float(out.split("smoke=")[1]) - n_tr) < 1e-4
    assert abs(mass - r.gather_rho().sum()) < 1e-6


def _build_example(tmp_path, name):
    exe = tmp_path / name
    lib = ROOT / "paper_2101_11856_b200" / "_build"
    subprocess.run(["g++", "-std=c++17", "-Wall", "-Werror", f"-I{ROOT / 'include'}",
                    str(ROOT / "examples" / f"{name}.cpp"), f"-L{lib}", "-llbmg", f"-Wl,-rpath,{lib}", "-o",
                    str(exe)], check=True)
    return exe


def test_cpp_tune_snapshot_example_compiles(tmp_path):
    assert _build_example(tmp_path, "tune_and_snapshot").exists()


@pytest.mark.gpu
def test_cpp_tune_snapshot_example_runs(tmp_path):
    exe = _build_example(tmp_path, "tune_and_snapshot")
    res = subprocess.run([str(exe), str(tmp_path)], capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    assert "tuned rows=6" in res.stdout and "last_snapshot=30 steps=30" in res.stdout
    import numpy as np
    from oracle import refpy
    for t in (10, 20, 30):
        dims, beta, rho = refpy.ref_load_field(tmp_path / f"rho_{t}.lbf", 32 * 24 * 24)
        assert dims == (32, 24, 24) and beta == 1 and abs(rho.mean() - 1.0) < 1e-2


def test_cpp_unit_calls_example_compiles(tmp_path):
    assert _build_example(tmp_path, "unit_calls").exists()


@pytest.mark.gpu
def test_cpp_unit_calls_example_runs(tmp_path):
    exe = _build_example(tmp_path, "unit_calls")
    res = subprocess.run([str(exe)], capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    out = res.stdout
    assert "step ok=1 t=8 max_df=0.000e+00" in out, out
    uerr = float(out.split("uerr=")[1].split()[0])
    spread = float(out.split("spread_err=")[1].split()[0])
    react = float(out.split("reaction_err=")[1].split()[0])
    assert "ib samples=64" in out and uerr <= 1e-15 and spread <= 1e-12 and react <= 1e-12, out
    assert "devices regions=2 dev1=0 max_drho=0.000e+00" in out, out
