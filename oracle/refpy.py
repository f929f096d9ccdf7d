"""TEST INFRASTRUCTURE ONLY (checker, never the measured path).

ctypes loader for the two CPU checkers built by oracle/Makefile:
  * oracle/_ref/libref_adapter.so — the unmodified reference compiled from
    /root/reference/proj/src (-Dlbm=lbm_ref) + ref_adapter.cpp
  * oracle/_build/liboracle.so    — the plain-C FP64 restatement
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs use it.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from paper_2101_11856_b200 import _abi
from paper_2101_11856_b200.scene import SceneConfig

HERE = Path(__file__).resolve().parent
REF_LIB = HERE / "_ref" / "libref_adapter.so"
ORACLE_LIB = HERE / "_build" / "liboracle.so"

_ref = None


def ref_available() -> bool:
    return REF_LIB.exists()


def ref_lib():
    global _ref
    if _ref is not None:
        return _ref
    if not REF_LIB.exists():
        raise FileNotFoundError(f"{REF_LIB} missing: run `make -C oracle ref` where /root/reference exists")
    L = C.CDLL(str(REF_LIB))
    P, D, I, SZ = C.c_void_p, C.POINTER(C.c_double), C.c_int, C.c_size_t
    U32P, U8P = C.POINTER(C.c_uint32), C.POINTER(C.c_uint8)
    CFG = C.POINTER(_abi.SceneConfigC)
    sig = {
        "ref_last_error": (C.c_char_p, []),
        "ref_runner_create": (I, [CFG, I, C.c_uint, C.POINTER(P)]),
        "ref_runner_create_with_samples": (I, [CFG, I, C.c_uint, C.POINTER(SZ), C.POINTER(D), C.POINTER(D),
                                               C.POINTER(U32P), C.POINTER(P)]),
        "ref_runner_destroy": (None, [P]),
        "ref_runner_create_tracers": (I, [CFG, I, C.c_uint, I, C.POINTER(_abi.EmitterC), C.POINTER(P)]),
        "ref_runner_tracer_count": (SZ, [P]),
        "ref_runner_tracers": (None, [P, D, C.POINTER(C.c_int64)]),
        "ref_emit_tracers": (SZ, [I, C.POINTER(_abi.EmitterC), C.c_long, C.c_uint64, D]),
        "ref_rasterize_density": (None, [SZ, D, I, I, I, D]),
        "ref_runner_advance": (I, [P, C.c_long, C.POINTER(_abi.StatusC)]),
        "ref_runner_advance_timed": (I, [P, C.c_long, C.POINTER(_abi.StatusC), C.POINTER(_abi.TimingRowC), SZ,
                                         C.POINTER(SZ)]),
        "ref_runner_step_count": (C.c_long, [P]),
        "ref_runner_set_layout": (I, [P, I, SZ]),
        "ref_runner_gather_rho": (None, [P, D]),
        "ref_runner_gather_u": (None, [P, D]),
        "ref_runner_gather_f": (None, [P, D]),
        "ref_runner_totals_count": (SZ, [P]),
        "ref_runner_totals": (None, [P, D]),
        "ref_runner_solid_count": (I, [P]),
        "ref_runner_sample_count": (SZ, [P, I, I]),
        "ref_runner_samples": (None, [P, I, I, D, D, D, D, D, U32P, U8P]),
        "ref_scene_sample_count": (SZ, [P, I]),
        "ref_scene_samples": (None, [P, I, D, D, U32P, D, C.POINTER(I), D]),
        "ref_make_rates": (I, [CFG, D]),
        "ref_collide_batch": (I, [CFG, SZ, D, D, D, D]),
        "ref_dense_collide_batch": (I, [CFG, SZ, D, D, D, D]),
        "ref_equilibrium": (None, [C.c_double, D, D]),
        "ref_lattice": (None, [C.POINTER(I), D, C.POINTER(I)]),
        "ref_moment_exponents": (None, [C.POINTER(I), C.POINTER(I)]),
        "ref_morton3": (C.c_uint64, [C.c_uint32, C.c_uint32, C.c_uint32]),
        "ref_split_domain": (I, [I, I, C.POINTER(I)]),
        "ref_face_owner": (None, [CFG, U8P]),
        "ref_reorder_permutation": (I, [SZ, D, U32P, I, U32P]),
        "ref_kernel_support": (I, [D, I, I, I, C.POINTER(I), D]),
        "ref_step": (I, [CFG, D, D, C.c_long, C.c_long, D, D, D, C.POINTER(_abi.StatusC)]),
        "ref_ib_interpolate_velocity": (I, [SZ, D, D, I, I, I, D, U8P]),
        "ref_ib_penalty_forces": (I, [SZ, D, D, D, U8P, D, I, I, I, D]),
        "ref_ib_spread_forces": (I, [SZ, D, D, U8P, I, I, I, I, D]),
        "ref_ib_update_rigid_motion": (I, [SZ, D, D, D, D, C.c_long, I, I, I, D, D, U8P]),
        "ref_ib_reaction_totals": (I, [SZ, D, D, D, I, I, D]),
        "ref_stream_and_faces": (I, [CFG, D, D]),
        "ref_gather_forces": (I, [SZ, D, D, U8P, I, I, I, D, U32P]),
        "ref_tune_spec": (I, [P, I, I, C.POINTER(I), C.POINTER(I), C.POINTER(SZ), SZ, C.POINTER(SZ)]),
        "ref_search_with_cost": (I, [I, I, C.POINTER(SZ), SZ, D, C.POINTER(I), C.POINTER(SZ), D]),
        "ref_dump_field": (I, [C.c_char_p, I, I, I, I, D]),
        "ref_load_field": (I, [C.c_char_p, C.POINTER(I), C.POINTER(I), D, SZ]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _ref = L
    return L


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _u32(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


def _u8(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def _check(code):
    if code:
        raise RuntimeError("reference: " + ref_lib().ref_last_error().decode())


def _emitters(emitters):
    arr = (_abi.EmitterC * max(len(emitters), 1))()
    for k, e in enumerate(emitters):
        arr[k].lo[:] = [float(v) for v in e.lo]
        arr[k].hi[:] = [float(v) for v in e.hi]
        arr[k].rate = int(e.rate)
    return arr


def ref_emit_tracers(emitters, step, seed):
    n = sum(int(e.rate) for e in emitters)
    out = np.zeros((n, 3))
    got = ref_lib().ref_emit_tracers(len(emitters), _emitters(emitters), step, seed, _dp(out))
    assert got == n
    return out


def ref_rasterize_density(positions, dims):
    pos = np.ascontiguousarray(positions, dtype=np.float64)
    nx, ny, nz = dims
    vol = np.zeros(nx * ny * nz)
    ref_lib().ref_rasterize_density(len(pos), _dp(pos), nx, ny, nz, _dp(vol))
    return vol


class RefRunner:
    """lbm_ref::Runner (the unmodified reference) driven through the adapter."""

    def __init__(self, cfg: SceneConfig, regions: int | None = None, threads: int | None = None,
                 samples: list | None = None):
        self.cfg = cfg
        L = ref_lib()
        cs = cfg.to_c()
        h = C.c_void_p()
        m = cfg.regions if regions is None else regions
        t = (os.cpu_count() or 1) if threads is None else threads
        if samples is None and cfg.emitters:
            em = _emitters(cfg.emitters)
            _check(L.ref_runner_create_tracers(cs.ptr, m, t, len(cfg.emitters), em, C.byref(h)))
        elif samples is None:
            _check(L.ref_runner_create(cs.ptr, m, t, C.byref(h)))
        else:
            ns = len(samples)
            keep = []
            counts = (C.c_size_t * ns)()
            pos = (C.POINTER(C.c_double) * ns)()
            refs = (C.POINTER(C.c_double) * ns)()
            srcs = (C.POINTER(C.c_uint32) * ns)()
            for k, s in enumerate(samples):
                p = np.ascontiguousarray(s["positions"], dtype=np.float64)
                r = np.ascontiguousarray(s["reference_positions"], dtype=np.float64)
                q = np.ascontiguousarray(s["source_id"], dtype=np.uint32)
                keep += [p, r, q]
                counts[k] = len(q)
                pos[k], refs[k], srcs[k] = _dp(p), _dp(r), _u32(q)
            _check(L.ref_runner_create_with_samples(cs.ptr, m, t, counts, pos, refs, srcs, C.byref(h)))
        self._h = h
        self.n = cfg.nx * cfg.ny * cfg.nz

    def __del__(self):
        if getattr(self, "_h", None):
            ref_lib().ref_runner_destroy(self._h)
            self._h = None

    def advance(self, steps: int):
        st = _abi.StatusC()
        _check(ref_lib().ref_runner_advance(self._h, steps, C.byref(st)))
        return {"ok": bool(st.ok), "mach_warning": bool(st.mach_warning), "step": int(st.step),
                "reason": st.reason.decode()}

    def advance_timed(self, steps: int):
        st = _abi.StatusC()
        cap = 16 * max(1, steps)
        rows = (_abi.TimingRowC * cap)()
        n = C.c_size_t()
        _check(ref_lib().ref_runner_advance_timed(self._h, steps, C.byref(st), rows, cap, C.byref(n)))
        return [(rows[k].phase.decode(), rows[k].step, rows[k].seconds) for k in range(n.value)]

    def step_count(self):
        return int(ref_lib().ref_runner_step_count(self._h))

    def tracers(self):
        n = ref_lib().ref_runner_tracer_count(self._h)
        pos = np.zeros((n, 3))
        birth = np.zeros(n, dtype=np.int64)
        ref_lib().ref_runner_tracers(self._h, _dp(pos), birth.ctypes.data_as(C.POINTER(C.c_int64)))
        return pos, birth

    def set_layout(self, ell, alpha):
        _check(ref_lib().ref_runner_set_layout(self._h, ell, alpha))

    def gather_rho(self):
        o = np.empty(self.n)
        ref_lib().ref_runner_gather_rho(self._h, _dp(o))
        return o

    def gather_u(self):
        o = np.empty((self.n, 3))
        ref_lib().ref_runner_gather_u(self._h, _dp(o))
        return o

    def gather_f(self):
        o = np.empty((self.n, 27))
        ref_lib().ref_runner_gather_f(self._h, _dp(o))
        return o

    def totals_log(self):
        n = ref_lib().ref_runner_totals_count(self._h)
        o = np.zeros((n, 6))
        if n:
            ref_lib().ref_runner_totals(self._h, _dp(o))
        return o

    def samples(self, region, solid):
        L = ref_lib()
        n = L.ref_runner_sample_count(self._h, region, solid)
        a = {k: np.zeros((n, 3)) for k in ("positions", "boundary_velocity", "penalty_force",
                                            "sampled_velocity", "reference_positions")}
        src = np.zeros(n, dtype=np.uint32)
        fl = np.zeros(n, dtype=np.uint8)
        L.ref_runner_samples(self._h, region, solid, _dp(a["positions"]), _dp(a["boundary_velocity"]),
                             _dp(a["penalty_force"]), _dp(a["sampled_velocity"]), _dp(a["reference_positions"]),
                             _u32(src), _u8(fl))
        a["source_id"] = src
        a["flagged"] = fl
        return a

    def scene_samples(self, solid):
        L = ref_lib()
        n = L.ref_scene_sample_count(self._h, solid)
        pos, ref = np.zeros((n, 3)), np.zeros((n, 3))
        src = np.zeros(n, dtype=np.uint32)
        bbox, rep = np.zeros(6), np.zeros(6)
        ell = C.c_int()
        L.ref_scene_samples(self._h, solid, _dp(pos), _dp(ref), _u32(src), _dp(bbox), C.byref(ell), _dp(rep))
        return {"positions": pos, "reference_positions": ref, "source_id": src, "bbox_lo": bbox[:3],
                "bbox_hi": bbox[3:], "block_edge": ell.value, "report": rep}


def ref_tune_spec(runner: "RefRunner", n_steps=10, warmup=5):
    L = ref_lib()
    lo, hi, n = C.c_int(), C.c_int(), C.c_size_t()
    buf = (C.c_size_t * 64)()
    _check(L.ref_tune_spec(runner._h, n_steps, warmup, C.byref(lo), C.byref(hi), buf, 64, C.byref(n)))
    return lo.value, hi.value, [int(buf[k]) for k in range(n.value)]


def ref_search_with_cost(ell_min, ell_max, alphas, table):
    L = ref_lib()
    a = (C.c_size_t * len(alphas))(*alphas)
    t = np.ascontiguousarray(table, dtype=np.float64)
    ell, alpha, best = C.c_int(), C.c_size_t(), C.c_double()
    _check(L.ref_search_with_cost(ell_min, ell_max, a, len(alphas), _dp(t), C.byref(ell), C.byref(alpha),
                                  C.byref(best)))
    return ell.value, alpha.value, best.value


def ref_dump_field(path, dims, field):
    a = np.ascontiguousarray(field, dtype=np.float64)
    nx, ny, nz = dims
    _check(ref_lib().ref_dump_field(str(path).encode(), nx, ny, nz, a.size // (nx * ny * nz), _dp(a)))


def ref_load_field(path, cap):
    d = (C.c_int * 3)()
    b = C.c_int()
    out = np.zeros(cap)
    _check(ref_lib().ref_load_field(str(path).encode(), d, C.byref(b), _dp(out), cap))
    return (d[0], d[1], d[2]), b.value, out


def ref_rates(cfg: SceneConfig):
    out = np.zeros(27)
    _check(ref_lib().ref_make_rates(cfg.to_c().ptr, _dp(out)))
    return out


def ref_collide(cfg: SceneConfig, f, rho, u, dense=False):
    f = np.ascontiguousarray(f, dtype=np.float64)
    rho = np.ascontiguousarray(rho, dtype=np.float64)
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.zeros_like(f)
    fn = ref_lib().ref_dense_collide_batch if dense else ref_lib().ref_collide_batch
    _check(fn(cfg.to_c().ptr, len(rho), _dp(f), _dp(rho), _dp(u), _dp(out)))
    return out


def ref_equilibrium(rho, u):
    out = np.zeros(27)
    uu = np.ascontiguousarray(u, dtype=np.float64)
    ref_lib().ref_equilibrium(rho, _dp(uu), _dp(out))
    return out


def ref_lattice():
    c = (C.c_int * 81)()
    w = np.zeros(27)
    opp = (C.c_int * 27)()
    ref_lib().ref_lattice(c, _dp(w), opp)
    return np.array(c[:], dtype=int).reshape(27, 3), w, np.array(opp[:], dtype=int)


def ref_moment_exponents():
    q = (C.c_int * 81)()
    d = (C.c_int * 27)()
    ref_lib().ref_moment_exponents(q, d)
    return np.array(q[:], dtype=int).reshape(27, 3), np.array(d[:], dtype=int)


def ref_morton3(x, y, z):
    return int(ref_lib().ref_morton3(x, y, z))


def ref_split_domain(nz, m):
    buf = (C.c_int * (2 * m))()
    _check(ref_lib().ref_split_domain(nz, m, buf))
    return [(buf[2 * r], buf[2 * r + 1]) for r in range(m)]


def ref_face_owner(cfg: SceneConfig):
    out = np.zeros((cfg.nx * cfg.ny * cfg.nz, 27), dtype=np.uint8)
    ref_lib().ref_face_owner(cfg.to_c().ptr, _u8(out))
    return out


def ref_reorder_permutation(positions, source_id, ell):
    pos = np.ascontiguousarray(positions, dtype=np.float64)
    src = np.ascontiguousarray(source_id, dtype=np.uint32)
    perm = np.zeros(len(src), dtype=np.uint32)
    _check(ref_lib().ref_reorder_permutation(len(src), _dp(pos), _u32(src), ell, _u32(perm)))
    return perm


def ref_kernel_support(pos, dims):
    p = np.ascontiguousarray(pos, dtype=np.float64)
    base = (C.c_int * 3)()
    w = np.zeros(6)
    inside = ref_lib().ref_kernel_support(_dp(p), dims[0], dims[1], dims[2], base, _dp(w))
    return bool(inside), tuple(base[:]), w


def ref_stream_and_faces(cfg: SceneConfig, f_prev, f_star):
    fp = np.ascontiguousarray(f_prev, dtype=np.float64)
    fs = np.array(f_star, dtype=np.float64, copy=True, order="C")
    _check(ref_lib().ref_stream_and_faces(cfg.to_c().ptr, _dp(fp), _dp(fs)))
    return fs


def ref_gather_forces(positions, forces, dims, flagged=None):
    pos = np.ascontiguousarray(positions, dtype=np.float64)
    frc = np.ascontiguousarray(forces, dtype=np.float64)
    n = len(pos)
    fl = np.zeros(n, dtype=np.uint8) if flagged is None else np.ascontiguousarray(flagged, dtype=np.uint8)
    N = dims[0] * dims[1] * dims[2]
    g = np.zeros((N, 3))
    loops = np.zeros(N, dtype=np.uint32)
    _check(ref_lib().ref_gather_forces(n, _dp(pos), _dp(frc), _u8(fl), dims[0], dims[1], dims[2], _dp(g),
                                       _u32(loops)))
    return g, loops


# ---- plain-C restatement (oracle/lbm_oracle.c) ------------------------------
_orc = None


def oracle_lib():
    global _orc
    if _orc is not None:
        return _orc
    if not ORACLE_LIB.exists():
        raise FileNotFoundError(f"{ORACLE_LIB} missing: run `make -C oracle oracle`")
    L = C.CDLL(str(ORACLE_LIB))
    P, D, I, SZ = C.c_void_p, C.POINTER(C.c_double), C.c_int, C.c_size_t
    U32P, U8P = C.POINTER(C.c_uint32), C.POINTER(C.c_uint8)
    CFG = C.POINTER(_abi.SceneConfigC)
    sig = {
        "orc_lattice": (None, [C.POINTER(I), D, C.POINTER(I), C.POINTER(I)]),
        "orc_make_rates": (I, [CFG, D]),
        "orc_equilibrium": (None, [C.c_double, D, D]),
        "orc_collide_batch": (I, [CFG, SZ, D, D, D, D]),
        "orc_morton3": (C.c_uint64, [C.c_uint32, C.c_uint32, C.c_uint32]),
        "orc_reorder_permutation": (I, [SZ, D, U32P, I, U32P]),
        "orc_split_domain": (I, [I, I, C.POINTER(I)]),
        "orc_face_owner": (None, [CFG, U8P]),
        "orc_kernel_support": (I, [D, I, I, I, C.POINTER(I), D]),
        "orc_create": (P, [CFG, C.POINTER(SZ), C.POINTER(D), C.POINTER(D), C.POINTER(U32P)]),
        "orc_destroy": (None, [P]),
        "orc_advance": (I, [P, C.c_long, C.POINTER(_abi.StatusC)]),
        "orc_step_count": (C.c_long, [P]),
        "orc_gather": (None, [P, I, D]),
        "orc_totals_count": (SZ, [P]),
        "orc_totals": (None, [P, D]),
        "orc_samples": (None, [P, I, D, D, D, D, U8P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _orc = L
    return L


class OracleRunner:
    """Single-region FP64 restatement (oracle/lbm_oracle.c).  Samples are
    passed in (storage order) so the oracle never re-implements sampling."""

    def __init__(self, cfg: SceneConfig, samples: list | None = None):
        L = oracle_lib()
        self.cfg = cfg
        self._cs = cfg.to_c()
        ns = len(cfg.solids)
        samples = samples or []
        if len(samples) != ns:
            raise ValueError("one sample set per solid is required")
        self._keep = []
        counts = (C.c_size_t * max(ns, 1))()
        pos = (C.POINTER(C.c_double) * max(ns, 1))()
        refs = (C.POINTER(C.c_double) * max(ns, 1))()
        srcs = (C.POINTER(C.c_uint32) * max(ns, 1))()
        for k, s in enumerate(samples):
            p = np.ascontiguousarray(s["positions"], dtype=np.float64)
            r = np.ascontiguousarray(s["reference_positions"], dtype=np.float64)
            q = np.ascontiguousarray(s["source_id"], dtype=np.uint32)
            self._keep += [p, r, q]
            counts[k] = len(q)
            pos[k], refs[k], srcs[k] = _dp(p), _dp(r), _u32(q)
        h = L.orc_create(self._cs.ptr, counts, pos, refs, srcs)
        if not h:
            raise ValueError("oracle: invalid collision model")
        self._h = h
        self.n = cfg.nx * cfg.ny * cfg.nz

    def __del__(self):
        if getattr(self, "_h", None):
            oracle_lib().orc_destroy(self._h)
            self._h = None

    def advance(self, steps):
        st = _abi.StatusC()
        oracle_lib().orc_advance(self._h, steps, C.byref(st))
        return {"ok": bool(st.ok), "mach_warning": bool(st.mach_warning), "step": int(st.step),
                "reason": st.reason.decode()}

    def step_count(self):
        return int(oracle_lib().orc_step_count(self._h))

    def _g(self, what, shape):
        o = np.empty(shape)
        oracle_lib().orc_gather(self._h, what, _dp(o))
        return o

    def gather_rho(self):
        return self._g(0, (self.n,))

    def gather_u(self):
        return self._g(1, (self.n, 3))

    def gather_f(self):
        return self._g(2, (self.n, 27))

    def totals_log(self):
        n = oracle_lib().orc_totals_count(self._h)
        o = np.zeros((n, 6))
        if n:
            oracle_lib().orc_totals(self._h, _dp(o))
        return o

    def samples(self, solid):
        n = len(self._keep[3 * solid + 2])
        a = {k: np.zeros((n, 3)) for k in ("positions", "boundary_velocity", "penalty_force", "sampled_velocity")}
        fl = np.zeros(n, dtype=np.uint8)
        oracle_lib().orc_samples(self._h, solid, _dp(a["positions"]), _dp(a["boundary_velocity"]),
                                 _dp(a["penalty_force"]), _dp(a["sampled_velocity"]), _u8(fl))
        a["flagged"] = fl
        return a


def oracle_collide(cfg: SceneConfig, f, rho, u):
    f = np.ascontiguousarray(f, dtype=np.float64)
    rho = np.ascontiguousarray(rho, dtype=np.float64)
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.zeros_like(f)
    if oracle_lib().orc_collide_batch(cfg.to_c().ptr, len(rho), _dp(f), _dp(rho), _dp(u), _dp(out)):
        raise ValueError("oracle: invalid collision model")
    return out


def oracle_face_owner(cfg: SceneConfig):
    out = np.zeros((cfg.nx * cfg.ny * cfg.nz, 27), dtype=np.uint8)
    oracle_lib().orc_face_owner(cfg.to_c().ptr, _u8(out))
    return out


def oracle_reorder_permutation(positions, source_id, ell):
    pos = np.ascontiguousarray(positions, dtype=np.float64)
    src = np.ascontiguousarray(source_id, dtype=np.uint32)
    perm = np.zeros(len(src), dtype=np.uint32)
    oracle_lib().orc_reorder_permutation(len(src), _dp(pos), _u32(src), ell, _u32(perm))
    return perm


def oracle_split_domain(nz, m):
    buf = (C.c_int * (2 * m))()
    if oracle_lib().orc_split_domain(nz, m, buf):
        raise ValueError("bad split")
    return [(buf[2 * r], buf[2 * r + 1]) for r in range(m)]


def ref_step(cfg: SceneConfig, f, f_star, t, steps):
    """lbm::step on an explicit single-region SimState: (f, rho, u, status)."""
    fa = np.ascontiguousarray(f, dtype=np.float64)
    fs = np.ascontiguousarray(f_star, dtype=np.float64)
    n = fa.size // 27
    fo, ro, uo = np.zeros((n, 27)), np.zeros(n), np.zeros((n, 3))
    st = _abi.StatusC()
    _check(ref_lib().ref_step(cfg.to_c().ptr, _dp(fa), _dp(fs), t, steps, _dp(fo), _dp(ro), _dp(uo), C.byref(st)))
    return fo, ro, uo, {"ok": bool(st.ok), "mach_warning": bool(st.mach_warning), "step": int(st.step),
                        "reason": st.reason.decode()}


def _a3(a):
    return np.ascontiguousarray(a, dtype=np.float64).reshape(-1, 3)


def ref_ib_interpolate_velocity(positions, u, dims):
    pos = _a3(positions)
    out = np.zeros((len(pos), 3))
    fl = np.zeros(len(pos), dtype=np.uint8)
    _check(ref_lib().ref_ib_interpolate_velocity(len(pos), _dp(pos), _dp(np.ascontiguousarray(u, dtype=np.float64)),
                                                 *dims, _dp(out), _u8(fl)))
    return out, fl


def ref_ib_penalty_forces(positions, ub, sampled, flagged, rho, dims):
    pos = _a3(positions)
    out = np.zeros((len(pos), 3))
    _check(ref_lib().ref_ib_penalty_forces(len(pos), _dp(pos), _dp(_a3(ub)), _dp(_a3(sampled)),
                                           _u8(np.ascontiguousarray(flagged, dtype=np.uint8)),
                                           _dp(np.ascontiguousarray(rho, dtype=np.float64)), *dims, _dp(out)))
    return out


def ref_ib_spread_forces(positions, force, flagged, g, dims, deterministic=False):
    pos = _a3(positions)
    out = np.array(g, dtype=np.float64, copy=True, order="C").reshape(-1, 3)
    _check(ref_lib().ref_ib_spread_forces(len(pos), _dp(pos), _dp(_a3(force)),
                                          _u8(np.ascontiguousarray(flagged, dtype=np.uint8)), *dims,
                                          int(deterministic), _dp(out)))
    return out


def ref_ib_update_rigid_motion(reference_positions, motion, t, dims):
    ref = _a3(reference_positions)
    n = len(ref)
    pos, ub, fl = np.zeros((n, 3)), np.zeros((n, 3)), np.zeros(n, dtype=np.uint8)
    v = np.ascontiguousarray(motion.linear_velocity, dtype=np.float64)
    w = np.ascontiguousarray(motion.angular_velocity, dtype=np.float64)
    c = np.ascontiguousarray(motion.center, dtype=np.float64)
    _check(ref_lib().ref_ib_update_rigid_motion(n, _dp(ref), _dp(v), _dp(w), _dp(c), t, *dims, _dp(pos), _dp(ub),
                                                _u8(fl)))
    return pos, ub, fl


def ref_ib_reaction_totals(positions, force, center, z0, z1):
    out = np.zeros(6)
    pos = _a3(positions)
    _check(ref_lib().ref_ib_reaction_totals(len(pos), _dp(pos), _dp(_a3(force)),
                                            _dp(np.ascontiguousarray(center, dtype=np.float64)), z0, z1, _dp(out)))
    return out[:3], out[3:]
