"""Python mirror of the reference's Runner / build_scene API over the C ABI.

Every call goes through the in-tree sm_100a library `_build/liblbmg.so`
(include/lbmg.h).  There is no CPU fallback: if the library is missing the
import fails loudly, and every device call raises when CUDA is unavailable.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from pathlib import Path
from typing import List, Optional

import numpy as np

from . import _abi
from .scene import ConfigError, SceneConfig

_LIB_PATH = Path(__file__).resolve().parent / "_build" / "liblbmg.so"
_lib = None


class LbmError(RuntimeError):
    pass


class CudaError(LbmError):
    pass


class StateError(LbmError):
    pass


def lib():
    """Load liblbmg.so (built by paper_2101_11856_b200/build.py)."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        raise ImportError(f"{_LIB_PATH} is missing: run `python -m paper_2101_11856_b200.build` "
                          "(the engine has no CPU fallback)")
    L = C.CDLL(str(_LIB_PATH))
    P, D, I, SZ = C.c_void_p, C.POINTER(C.c_double), C.c_int, C.c_size_t
    U32P, U8P = C.POINTER(C.c_uint32), C.POINTER(C.c_uint8)
    sig = {
        "lbmg_abi_version": (I, []),
        "lbmg_last_error": (C.c_char_p, []),
        "lbmg_device_count": (I, []),
        "lbmg_scene_config_default": (None, [C.POINTER(_abi.SceneConfigC)]),
        "lbmg_validate_config": (I, [C.POINTER(_abi.SceneConfigC), D]),
        "lbmg_scene_build": (I, [C.POINTER(_abi.SceneConfigC), C.POINTER(P)]),
        "lbmg_scene_destroy": (None, [P]),
        "lbmg_scene_solid_count": (I, [P]),
        "lbmg_scene_sample_count": (SZ, [P, I]),
        "lbmg_scene_samples": (I, [P, I, D, D, U32P, U8P, D, C.POINTER(I)]),
        "lbmg_scene_set_samples": (I, [P, I, SZ, D, D, U32P]),
        "lbmg_morton3": (C.c_uint64, [C.c_uint32, C.c_uint32, C.c_uint32]),
        "lbmg_reorder_permutation": (I, [SZ, D, U32P, I, U32P]),
        "lbmg_split_domain": (I, [I, I, C.POINTER(I)]),
        "lbmg_runner_create": (I, [P, I, I, C.POINTER(P)]),
        "lbmg_runner_create_rank": (I, [P, I, I, I, C.POINTER(P)]),
        "lbmg_runner_create_devices": (I, [P, I, I, C.POINTER(I), C.POINTER(P)]),
        "lbmg_runner_region_device": (I, [P, I]),
        "lbmg_runner_destroy": (None, [P]),
        "lbmg_runner_clone": (I, [P, C.POINTER(P)]),
        "lbmg_runner_set_stream": (I, [P, P]),
        "lbmg_runner_advance": (I, [P, C.c_long, C.POINTER(_abi.StatusC), C.POINTER(_abi.TimingRowC), SZ,
                                    C.POINTER(SZ)]),
        "lbmg_runner_step_count": (C.c_long, [P]),
        "lbmg_runner_status": (I, [P, C.POINTER(_abi.StatusC)]),
        "lbmg_runner_dims": (I, [P, C.POINTER(I), C.POINTER(I), C.POINTER(I)]),
        "lbmg_runner_region_count": (I, [P]),
        "lbmg_runner_set_layout": (I, [P, I, SZ]),
        "lbmg_runner_alpha": (SZ, [P]),
        "lbmg_runner_set_variant": (I, [P, I, I]),
        "lbmg_runner_variant": (I, [P, C.POINTER(I), C.POINTER(I)]),
        "lbmg_runner_measure_cost": (I, [P, I, SZ, I, I, C.POINTER(C.c_double)]),
        "lbmg_runner_layout_key": (I, [P, SZ, C.POINTER(C.c_uint64)]),
        "lbmg_runner_block_edge": (I, [P]),
        "lbmg_runner_gather_rho": (I, [P, D]),
        "lbmg_runner_gather_u": (I, [P, D]),
        "lbmg_runner_gather_f": (I, [P, D]),
        "lbmg_runner_snapshot_begin": (I, [P]),
        "lbmg_runner_snapshot_wait": (I, [P, D, D, C.POINTER(C.c_long)]),
        "lbmg_dump_field": (I, [C.c_char_p, I, I, I, I, D]),
        "lbmg_runner_slab": (I, [P, C.POINTER(I), C.POINTER(I)]),
        "lbmg_runner_totals_count": (SZ, [P]),
        "lbmg_runner_totals": (I, [P, D, SZ]),
        "lbmg_runner_sample_count": (SZ, [P, I, I]),
        "lbmg_runner_samples": (I, [P, I, I, D, D, D, D, U32P, U8P]),
        "lbmg_runner_cell_flags": (I, [P, U8P]),
        "lbmg_runner_halo_f": (I, [P, I, C.POINTER(P), C.POINTER(P), C.POINTER(P), C.POINTER(P), C.POINTER(SZ)]),
        "lbmg_runner_halo_macro": (I, [P, C.POINTER(P), C.POINTER(P), C.POINTER(P), C.POINTER(P),
                                       C.POINTER(SZ)]),
        "lbmg_runner_phase": (I, [P, I, I]),
        "lbmg_runner_sync": (I, [P, C.POINTER(_abi.StatusC)]),
        "lbmg_collide_batch": (I, [C.POINTER(_abi.SceneConfigC), SZ, D, D, D, D]),
        "lbmg_step": (I, [P, C.POINTER(_abi.StatusC)]),
        "lbmg_runner_load_state": (I, [P, D, D, C.c_long]),
        "lbmg_ib_kernel_support": (I, [SZ, D, I, I, I, C.POINTER(I), D, U8P]),
        "lbmg_ib_interpolate_velocity": (I, [SZ, D, D, I, I, I, I, I, D, U8P]),
        "lbmg_ib_penalty_forces": (I, [SZ, D, D, D, U8P, D, I, I, I, I, I, D]),
        "lbmg_ib_spread_forces": (I, [SZ, D, D, U8P, I, I, I, I, I, D]),
        "lbmg_ib_update_rigid_motion": (I, [SZ, D, D, D, D, C.c_long, I, I, I, D, D, U8P]),
        "lbmg_ib_reaction_totals": (I, [SZ, D, D, D, I, I, D]),
        "lbmg_runner_kernels_per_step": (C.c_long, [P]),
        "lbmg_runner_sync_interval": (C.c_long, [P]),
        "lbmg_runner_kernel_launches": (C.c_long, [P]),
        "lbmg_runner_set_cta": (I, [P, I]),
        "lbmg_runner_cta": (I, [P]),
        "lbmg_scene_set_emitters": (I, [P, I, C.POINTER(_abi.EmitterC)]),
        "lbmg_emit_tracers": (I, [I, C.POINTER(_abi.EmitterC), C.c_long, C.c_uint64, D]),
        "lbmg_runner_tracer_count": (SZ, [P]),
        "lbmg_runner_tracers": (I, [P, D, C.POINTER(C.c_int64)]),
        "lbmg_runner_tracer_density": (I, [P, D]),
        "lbmg_rasterize_density": (I, [SZ, D, I, I, I, I, D]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def _check(code: int):
    if code == 0:
        return
    msg = lib().lbmg_last_error().decode(errors="replace")
    if code == 1:
        raise ConfigError(msg)
    if code in (2, 3):
        raise CudaError(msg)
    raise StateError(msg)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _u32(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


def _u8(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def dump_field(path, dims, field: np.ndarray):
    """LBF1 canonical field dump (io.cpp:34-55), readable by the reference's load_field."""
    a = np.ascontiguousarray(field, dtype=np.float64)
    nx, ny, nz = dims
    beta = a.size // (nx * ny * nz)
    if beta * nx * ny * nz != a.size:
        raise ConfigError("dump_field: field size does not match dims")
    _check(lib().lbmg_dump_field(str(path).encode(), nx, ny, nz, beta, _dp(a)))


def device_count() -> int:
    return lib().lbmg_device_count()


def model_rates(cfg: SceneConfig) -> np.ndarray:
    """Effective rates in canonical moment-row order (SceneConfig::make_model)."""
    cs = cfg.to_c()
    out = np.zeros(27)
    _check(lib().lbmg_validate_config(cs.ptr, _dp(out)))
    return out


def morton3(x: int, y: int, z: int) -> int:
    return int(lib().lbmg_morton3(x, y, z))


def reorder_permutation(positions: np.ndarray, source_id: np.ndarray, ell: int) -> np.ndarray:
    pos = np.ascontiguousarray(positions, dtype=np.float64)
    src = np.ascontiguousarray(source_id, dtype=np.uint32)
    perm = np.zeros(len(src), dtype=np.uint32)
    _check(lib().lbmg_reorder_permutation(len(src), _dp(pos), _u32(src), ell, _u32(perm)))
    return perm


def split_domain(nz: int, m: int) -> List[tuple]:
    buf = (C.c_int * (2 * max(m, 1)))()
    _check(lib().lbmg_split_domain(nz, m, buf))
    return [(buf[2 * r], buf[2 * r + 1]) for r in range(m)]


@dataclass
class StepStatus:
    ok: bool = True
    mach_warning: bool = False
    step: int = -1
    reason: str = ""

    @staticmethod
    def _from(c: _abi.StatusC) -> "StepStatus":
        return StepStatus(bool(c.ok), bool(c.mach_warning), int(c.step), c.reason.decode())


@dataclass
class TimingRow:
    phase: str
    step: int
    seconds: float


def _emitters_c(emitters):
    arr = (_abi.EmitterC * max(len(emitters), 1))()
    for k, e in enumerate(emitters):
        arr[k].lo[:] = [float(v) for v in e.lo]
        arr[k].hi[:] = [float(v) for v in e.hi]
        arr[k].rate = int(e.rate)
    return arr


@dataclass
class TracerCloud:
    """tracer.hpp:19-25: live particles in emission order (retired ones removed)."""
    positions: np.ndarray  # (n, 3) FP64
    birth_step: np.ndarray  # (n,) int64

    def size(self) -> int:
        return len(self.birth_step)


def emit_tracers(emitters, step: int, seed: int) -> np.ndarray:
    """emit_tracers (tracer.cpp:28-40): the positions step `step` appends, (E, 3)."""
    n = sum(int(e.rate) for e in emitters)
    out = np.zeros((n, 3))
    _check(lib().lbmg_emit_tracers(len(emitters), _emitters_c(emitters), step, seed, _dp(out)))
    return out


def rasterize_density(cloud, dims, device: int = 0) -> np.ndarray:
    """rasterize_density (tracer.cpp:67-92) on the device: (nz, ny, nx) flattened
    in node_index order, FP64."""
    pos = np.ascontiguousarray(cloud.positions if hasattr(cloud, "positions") else cloud, dtype=np.float64)
    nx, ny, nz = dims
    vol = np.zeros(nx * ny * nz)
    _check(lib().lbmg_rasterize_density(len(pos), _dp(pos), nx, ny, nz, device, _dp(vol)))
    return vol


class Scene:
    """build_scene (scene.cpp:341-366): sampled, ordered, motion-annotated solids."""

    def __init__(self, cfg: SceneConfig):
        self.cfg = cfg
        cs = cfg.to_c()
        h = C.c_void_p()
        _check(lib().lbmg_scene_build(cs.ptr, C.byref(h)))
        self._h = h
        if cfg.emitters:
            em = _emitters_c(cfg.emitters)
            _check(lib().lbmg_scene_set_emitters(h, len(cfg.emitters), em))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().lbmg_scene_destroy(self._h)
            self._h = None

    @property
    def solid_count(self) -> int:
        return lib().lbmg_scene_solid_count(self._h)

    def samples(self, solid: int) -> dict:
        n = lib().lbmg_scene_sample_count(self._h, solid)
        pos, ref = np.zeros((n, 3)), np.zeros((n, 3))
        src = np.zeros(n, dtype=np.uint32)
        bbox = np.zeros(6)
        ell = C.c_int()
        _check(lib().lbmg_scene_samples(self._h, solid, _dp(pos), _dp(ref), _u32(src), None, _dp(bbox),
                                        C.byref(ell)))
        return {"positions": pos, "reference_positions": ref, "source_id": src, "bbox_lo": bbox[:3],
                "bbox_hi": bbox[3:], "block_edge": ell.value}

    def set_samples(self, solid: int, positions, reference_positions, source_id):
        pos = np.ascontiguousarray(positions, dtype=np.float64)
        ref = np.ascontiguousarray(reference_positions, dtype=np.float64)
        src = np.ascontiguousarray(source_id, dtype=np.uint32)
        _check(lib().lbmg_scene_set_samples(self._h, solid, len(src), _dp(pos), _dp(ref), _u32(src)))


def build_scene(cfg: SceneConfig) -> Scene:
    return Scene(cfg)


class Runner:
    """lbm::Runner (runner.hpp:25-83) on the B200 engine."""

    def __init__(self, scene: Scene, regions: Optional[int] = None, device: int = 0, *,
                 world: int = 0, rank: int = 0, devices: Optional[List[int]] = None, _handle=None):
        """regions z-slabs in this process: on `device`, or — with `devices` —
        region r on devices[r % len(devices)] (peer-access halos, one stream
        per slab); world/rank: one slab of a multi-process run."""
        self.scene = scene
        if _handle is not None:
            self._h = _handle
            return
        h = C.c_void_p()
        if world > 0:
            _check(lib().lbmg_runner_create_rank(scene._h, world, rank, device, C.byref(h)))
        elif devices:
            m = scene.cfg.regions if regions is None else regions
            arr = (C.c_int * len(devices))(*devices)
            _check(lib().lbmg_runner_create_devices(scene._h, m, len(devices), arr, C.byref(h)))
        else:
            m = scene.cfg.regions if regions is None else regions
            _check(lib().lbmg_runner_create(scene._h, m, device, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().lbmg_runner_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    # -- stepping ----------------------------------------------------------
    def advance(self, steps: int, timings: Optional[list] = None) -> StepStatus:
        st = _abi.StatusC()
        if timings is None:
            _check(lib().lbmg_runner_advance(self._h, steps, C.byref(st), None, 0, None))
        else:
            cap = max(1, steps) * 5  # boundary, ib, fluid, tracers, total
            rows = (_abi.TimingRowC * cap)()
            n = C.c_size_t()
            _check(lib().lbmg_runner_advance(self._h, steps, C.byref(st), rows, cap, C.byref(n)))
            for k in range(n.value):
                timings.append(TimingRow(rows[k].phase.decode(), rows[k].step, rows[k].seconds))
        return StepStatus._from(st)

    def step(self) -> StepStatus:
        """step(SimState&, ...) (solver.hpp:82-83): one single-region step without solids."""
        st = _abi.StatusC()
        _check(lib().lbmg_step(self._h, C.byref(st)))
        return StepStatus._from(st)

    def load_state(self, f, f_star=None, t: int = 0):
        """The explicit SimState step() advances: f(t) (nodes x 27, FP64 AoS), the
        face-pass scratch f_star (seeds the persistent face slots; None: f), t."""
        fa = np.ascontiguousarray(f, dtype=np.float64)
        fs = None if f_star is None else np.ascontiguousarray(f_star, dtype=np.float64)
        if fa.size != self._n_local() * 27 or (fs is not None and fs.size != fa.size):
            raise ConfigError("load_state: f and f_star hold nodes x 27 values")
        _check(lib().lbmg_runner_load_state(self._h, _dp(fa), None if fs is None else _dp(fs), t))

    def step_count(self) -> int:
        return int(lib().lbmg_runner_step_count(self._h))

    def status(self) -> StepStatus:
        st = _abi.StatusC()
        _check(lib().lbmg_runner_status(self._h, C.byref(st)))
        return StepStatus._from(st)

    def dims(self):
        x, y, z = C.c_int(), C.c_int(), C.c_int()
        _check(lib().lbmg_runner_dims(self._h, C.byref(x), C.byref(y), C.byref(z)))
        return (x.value, y.value, z.value)

    def region_count(self) -> int:
        return lib().lbmg_runner_region_count(self._h)

    def region_device(self, region: int) -> int:
        return int(lib().lbmg_runner_region_device(self._h, region))

    def set_layout(self, block_edge: int, alpha: int):
        _check(lib().lbmg_runner_set_layout(self._h, block_edge, alpha))

    def alpha(self) -> int:
        return int(lib().lbmg_runner_alpha(self._h))

    def set_variant(self, fluid: int, ib: int, cta: Optional[int] = None):
        """Kernel variants (tuner launch-split dimension): fluid 0 = TMA-staged
        ghost-layout kernel, 1 = register-direct compact kernels; ib 0 = fused
        single-region IB kernel, 1 = split IB pipeline; cta = threads per CTA of
        the staged kernel (512/256/128, 0 = default; None keeps it)."""
        _check(lib().lbmg_runner_set_variant(self._h, fluid, ib))
        if cta is not None:
            self.set_cta(cta)

    def set_cta(self, threads: int):
        _check(lib().lbmg_runner_set_cta(self._h, threads))

    def cta(self) -> int:
        return int(lib().lbmg_runner_cta(self._h))

    def variant(self):
        f, i = C.c_int(), C.c_int()
        _check(lib().lbmg_runner_variant(self._h, C.byref(f), C.byref(i)))
        return f.value, i.value

    def measure_cost(self, block_edge: int, alpha: int, warmup: int, n_steps: int) -> float:
        """autotune.cpp:29-36 on the device: mean seconds per step (CUDA events), inf on divergence."""
        out = C.c_double()
        _check(lib().lbmg_runner_measure_cost(self._h, block_edge, alpha, warmup, n_steps, C.byref(out)))
        return out.value

    def layout_key(self, alpha: int) -> int:
        k = C.c_uint64()
        _check(lib().lbmg_runner_layout_key(self._h, alpha, C.byref(k)))
        return k.value

    def block_edge(self) -> int:
        return int(lib().lbmg_runner_block_edge(self._h))

    def clone(self) -> "Runner":
        h = C.c_void_p()
        _check(lib().lbmg_runner_clone(self._h, C.byref(h)))
        return Runner(self.scene, _handle=h)

    def set_stream(self, stream_ptr: int):
        _check(lib().lbmg_runner_set_stream(self._h, C.c_void_p(stream_ptr)))

    # -- readback ----------------------------------------------------------
    def slab(self):
        z0, z1 = C.c_int(), C.c_int()
        _check(lib().lbmg_runner_slab(self._h, C.byref(z0), C.byref(z1)))
        return z0.value, z1.value

    def _n_local(self):
        nx, ny, _ = self.dims()
        z0, z1 = self.slab()
        return nx * ny * (z1 - z0)

    def gather_rho(self) -> np.ndarray:
        out = np.empty(self._n_local())
        _check(lib().lbmg_runner_gather_rho(self._h, _dp(out)))
        return out

    def gather_u(self) -> np.ndarray:
        out = np.empty((self._n_local(), 3))
        _check(lib().lbmg_runner_gather_u(self._h, _dp(out)))
        return out

    def gather_f(self) -> np.ndarray:
        out = np.empty((self._n_local(), 27))
        _check(lib().lbmg_runner_gather_f(self._h, _dp(out)))
        return out


    def snapshot_begin(self):
        """Start an asynchronous rho*/u* snapshot of the current step (returns at once)."""
        _check(lib().lbmg_runner_snapshot_begin(self._h))

    def snapshot_wait(self):
        """(step, rho[N], u[N,3]) of the snapshot started by snapshot_begin."""
        nx, ny, nz = self.dims()
        z0, z1 = self.slab()
        n = nx * ny * (z1 - z0)
        rho, u = np.empty(n), np.empty((n, 3))
        t = C.c_long()
        _check(lib().lbmg_runner_snapshot_wait(self._h, _dp(rho), _dp(u), C.byref(t)))
        return t.value, rho, u
    def totals_log(self) -> np.ndarray:
        n = lib().lbmg_runner_totals_count(self._h)
        out = np.zeros((n, 6))
        if n:
            _check(lib().lbmg_runner_totals(self._h, _dp(out), n))
        return out

    def samples(self, region: int, solid: int) -> dict:
        n = lib().lbmg_runner_sample_count(self._h, region, solid)
        arrs = {k: np.zeros((n, 3)) for k in ("positions", "boundary_velocity", "penalty_force",
                                               "sampled_velocity")}
        src = np.zeros(n, dtype=np.uint32)
        fl = np.zeros(n, dtype=np.uint8)
        _check(lib().lbmg_runner_samples(self._h, region, solid, _dp(arrs["positions"]),
                                         _dp(arrs["boundary_velocity"]), _dp(arrs["penalty_force"]),
                                         _dp(arrs["sampled_velocity"]), _u32(src), _u8(fl)))
        arrs["source_id"] = src
        arrs["flagged"] = fl
        return arrs

    # -- tracers (runner.hpp:54, runner.cpp:213-223) -------------------------
    def tracers(self) -> TracerCloud:
        n = int(lib().lbmg_runner_tracer_count(self._h))
        pos = np.zeros((n, 3))
        birth = np.zeros(n, dtype=np.int64)
        _check(lib().lbmg_runner_tracers(self._h, _dp(pos), birth.ctypes.data_as(C.POINTER(C.c_int64))))
        return TracerCloud(pos, birth)

    def tracer_density(self) -> np.ndarray:
        """rasterize_density(tracers(), dims) from the device-resident cloud."""
        nx, ny, nz = self.dims()
        vol = np.zeros(nx * ny * nz)
        _check(lib().lbmg_runner_tracer_density(self._h, _dp(vol)))
        return vol

    def cell_flags(self) -> np.ndarray:
        out = np.zeros((self._n_local(), 27), dtype=np.uint8)
        _check(lib().lbmg_runner_cell_flags(self._h, _u8(out)))
        return out

    # -- rank mode (multi-process halo exchange) ---------------------------
    def halo_f(self, parity: int):
        ptrs = [C.c_void_p() for _ in range(4)]
        nb = C.c_size_t()
        _check(lib().lbmg_runner_halo_f(self._h, parity, *[C.byref(p) for p in ptrs], C.byref(nb)))
        return [p.value for p in ptrs], nb.value

    def halo_macro(self):
        ptrs = [C.c_void_p() for _ in range(4)]
        nb = C.c_size_t()
        _check(lib().lbmg_runner_halo_macro(self._h, *[C.byref(p) for p in ptrs], C.byref(nb)))
        return [p.value for p in ptrs], nb.value

    def phase(self, ph: int, write_macro: bool = False):
        _check(lib().lbmg_runner_phase(self._h, ph, int(write_macro)))

    def sync_interval(self) -> int:
        """Most steps between two sync() calls in an externally driven run."""
        return int(lib().lbmg_runner_sync_interval(self._h))

    def kernel_launches(self) -> int:
        """Engine kernels launched by advance() so far (graph kernel nodes included)."""
        return int(lib().lbmg_runner_kernel_launches(self._h))

    def kernels_per_step(self) -> int:
        return int(lib().lbmg_runner_kernels_per_step(self._h))

    def sync(self) -> StepStatus:
        st = _abi.StatusC()
        _check(lib().lbmg_runner_sync(self._h, C.byref(st)))
        return StepStatus._from(st)


def collide_batch(cfg: SceneConfig, f: np.ndarray, rho: np.ndarray, u: np.ndarray) -> np.ndarray:
    """collide() of n nodes on the device (fp32 arithmetic)."""
    f = np.ascontiguousarray(f, dtype=np.float64)
    rho = np.ascontiguousarray(rho, dtype=np.float64)
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.zeros_like(f)
    cs = cfg.to_c()
    _check(lib().lbmg_collide_batch(cs.ptr, len(rho), _dp(f), _dp(rho), _dp(u), _dp(out)))
    return out


# ---- the IB free functions (ib.hpp:77-128) on the device ------------------

def _v3(a):
    return np.ascontiguousarray(a, dtype=np.float64).reshape(-1, 3)


def _dims3(dims):
    nx, ny, nz = (int(v) for v in dims)
    return nx, ny, nz


def ib_kernel_support(positions, dims):
    """kernel_support (ib.cpp:294-308) per sample: (base (n,3) int32, w (n,6), inside (n,) bool)."""
    pos = _v3(positions)
    n = len(pos)
    base = np.zeros((n, 3), dtype=np.int32)
    w = np.zeros((n, 6))
    inside = np.zeros(n, dtype=np.uint8)
    _check(lib().lbmg_ib_kernel_support(n, _dp(pos), *_dims3(dims), base.ctypes.data_as(C.POINTER(C.c_int)), _dp(w),
                                        _u8(inside)))
    return base, w, inside.astype(bool)


def ib_interpolate_velocity(positions, u, dims, slab=None):
    """interpolate_velocity (ib.cpp:321-343): (sampled (n,3), flagged (n,) uint8)."""
    pos = _v3(positions)
    uu = np.ascontiguousarray(u, dtype=np.float64)
    nx, ny, nz = _dims3(dims)
    z0, z1 = slab or (0, nz)
    out = np.zeros((len(pos), 3))
    fl = np.zeros(len(pos), dtype=np.uint8)
    _check(lib().lbmg_ib_interpolate_velocity(len(pos), _dp(pos), _dp(uu), nx, ny, nz, z0, z1, _dp(out), _u8(fl)))
    return out, fl


def ib_penalty_forces(positions, boundary_velocity, sampled_velocity, flagged, rho, dims, slab=None):
    """penalty_forces (ib.cpp:345-365): rho(x_s) (u_b - u(x_s)), (n,3)."""
    pos = _v3(positions)
    ub, us = _v3(boundary_velocity), _v3(sampled_velocity)
    fl = np.ascontiguousarray(flagged, dtype=np.uint8)
    r = np.ascontiguousarray(rho, dtype=np.float64)
    nx, ny, nz = _dims3(dims)
    z0, z1 = slab or (0, nz)
    out = np.zeros((len(pos), 3))
    _check(lib().lbmg_ib_penalty_forces(len(pos), _dp(pos), _dp(ub), _dp(us), _u8(fl), _dp(r), nx, ny, nz, z0, z1,
                                        _dp(out)))
    return out


def ib_spread_forces(positions, penalty_force, flagged, g, dims, slab=None):
    """spread_forces (ib.cpp:369-454, atomic mode): returns g + the spread forces (nodes,3)."""
    pos = _v3(positions)
    fo = _v3(penalty_force)
    fl = np.ascontiguousarray(flagged, dtype=np.uint8)
    out = np.array(g, dtype=np.float64, copy=True, order="C").reshape(-1, 3)
    nx, ny, nz = _dims3(dims)
    z0, z1 = slab or (0, nz)
    _check(lib().lbmg_ib_spread_forces(len(pos), _dp(pos), _dp(fo), _u8(fl), nx, ny, nz, z0, z1, _dp(out)))
    return out


def ib_update_rigid_motion(reference_positions, motion, t, dims):
    """update_rigid_motion (ib.cpp:456-489): (positions, boundary_velocity, flagged) at step t."""
    ref = _v3(reference_positions)
    v = np.ascontiguousarray(motion.linear_velocity, dtype=np.float64)
    w = np.ascontiguousarray(motion.angular_velocity, dtype=np.float64)
    c = np.ascontiguousarray(motion.center, dtype=np.float64)
    n = len(ref)
    pos, ub = np.zeros((n, 3)), np.zeros((n, 3))
    fl = np.zeros(n, dtype=np.uint8)
    _check(lib().lbmg_ib_update_rigid_motion(n, _dp(ref), _dp(v), _dp(w), _dp(c), t, *_dims3(dims), _dp(pos), _dp(ub),
                                             _u8(fl)))
    return pos, ub, fl


def ib_reaction_totals(positions, penalty_force, center, z0, z1):
    """reaction_totals (ib.cpp:491-501): (force (3,), torque (3,))."""
    pos, fo = _v3(positions), _v3(penalty_force)
    c = np.ascontiguousarray(center, dtype=np.float64)
    out = np.zeros(6)
    _check(lib().lbmg_ib_reaction_totals(len(pos), _dp(pos), _dp(fo), _dp(c), z0, z1, _dp(out)))
    return out[:3], out[3:]
