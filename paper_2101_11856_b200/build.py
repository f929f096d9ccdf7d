"""In-tree build of the sm_100a engine: csrc/* -> _build/liblbmg.so.

nvcc cross-compiles for sm_100a without a GPU; the resulting .so travels to
the GPU box with the repo snapshot.  cudart is linked statically so the
library does not depend on a runtime search path.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "_build"
LIB = OUT / "liblbmg.so"

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = [
    "-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
    f"-I{ROOT / 'include'}", f"-I{CSRC}",
]
SOURCES = ["fluid.cu", "kernels.cu", "ib_free.cu", "tracers.cu", "scene.cpp", "runner.cpp", "capi.cpp"]


def _obj(src: str) -> Path:
    return OUT / (src + ".o")


def _stale(src: str) -> bool:
    obj = _obj(src)
    if not obj.exists():
        return True
    deps = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp")) + [CSRC / src, ROOT / "include" / "lbmg.h"]
    return any(d.stat().st_mtime > obj.stat().st_mtime for d in deps)


def _compile(src: str) -> str:
    cmd = [NVCC, *ARCH, *COMMON]
    if src.endswith(".cu"):
        cmd += ["-Xptxas", "-v"] if os.environ.get("LBMG_PTXAS_V") else []
    else:
        cmd += ["-x", "cu"] if False else []
    cmd += ["-c", str(CSRC / src), "-o", str(_obj(src))]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return r.stderr


def build(force: bool = False, verbose: bool = False) -> Path:
    OUT.mkdir(exist_ok=True)
    todo = [s for s in SOURCES if force or _stale(s)]
    if todo:
        with cf.ThreadPoolExecutor(max_workers=len(todo)) as ex:
            for src, log in zip(todo, ex.map(_compile, todo)):
                if verbose and log:
                    print(f"[{src}]\n{log}", file=sys.stderr)
    if todo or not LIB.exists() or any(_obj(s).stat().st_mtime > LIB.stat().st_mtime for s in SOURCES):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *[str(_obj(s)) for s in SOURCES], "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
