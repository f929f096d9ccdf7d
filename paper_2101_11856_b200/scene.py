"""Scene configuration: the Python face of SceneConfig (scene.hpp:49-78).

Field names, enum spellings and defaults follow the reference's C++ struct and
its strict JSON schema (scene.cpp:132-331), so a scene file written for the
reference loads unchanged (`parse_scene_config` / `load_scene_config`).
"""
from __future__ import annotations

import ctypes as C
import json
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

from . import _abi

KINDS = {"bgk": _abi.BGK, "rm-mrt": _abi.RAW_MRT, "cm-mrt": _abi.CENTRAL_MRT}
POLICIES = {"constant": _abi.POLICY_CONSTANT, "relax-toward-one": _abi.POLICY_RELAX_TOWARD_ONE}
CONDITIONS = {"no-slip": _abi.NOSLIP, "inlet": _abi.INLET, "outflow": _abi.OUTFLOW, "periodic": _abi.PERIODIC}
MESHES = {"sphere": _abi.MESH_SPHERE, "box": _abi.MESH_BOX, "fin-comb": _abi.MESH_FIN_COMB, "quad": _abi.MESH_QUAD}
SAMPLING = {"dart-throwing": _abi.SAMPLING_DART, "elimination": _abi.SAMPLING_ELIMINATION}
INITS = {"uniform": _abi.INIT_UNIFORM, "taylor-green": _abi.INIT_TAYLOR_GREEN}
IB_MODES = {"atomic": _abi.IB_ATOMIC, "deterministic": _abi.IB_DETERMINISTIC}
FACE_NAMES = ("x-", "x+", "y-", "y+", "z-", "z+")


class ConfigError(ValueError):
    """lbm::ConfigError (core.hpp:50-53)."""


@dataclass
class FaceSpec:
    condition: str = "no-slip"
    velocity: Sequence[float] = (0.0, 0.0, 0.0)


@dataclass
class MeshConfig:
    type: str = "sphere"
    center: Sequence[float] = (0.0, 0.0, 0.0)
    radius: float = 1.0
    subdivisions: int = 3
    lo: Sequence[float] = (0.0, 0.0, 0.0)
    hi: Sequence[float] = (0.0, 0.0, 0.0)
    origin: Sequence[float] = (0.0, 0.0, 0.0)
    fins: int = 8
    fin_length: float = 8.0
    fin_height: float = 6.0
    fin_spacing: float = 2.0
    size: float = 1.0
    plane_z: float = 0.0


@dataclass
class RigidMotion:
    linear_velocity: Sequence[float] = (0.0, 0.0, 0.0)
    angular_velocity: Sequence[float] = (0.0, 0.0, 0.0)
    center: Sequence[float] = (0.0, 0.0, 0.0)


@dataclass
class SolidConfig:
    mesh: MeshConfig = field(default_factory=MeshConfig)
    poisson_radius: float = 0.5
    sampling: str = "dart-throwing"
    motion: Optional[RigidMotion] = None


@dataclass
class TracerEmitter:
    """tracer.hpp:14-17: axis-aligned emission region (grid units), particles per step."""
    lo: Sequence[float] = (0.0, 0.0, 0.0)
    hi: Sequence[float] = (0.0, 0.0, 0.0)
    rate: int = 0


@dataclass
class SceneConfig:
    nx: int = 0
    ny: int = 0
    nz: int = 0
    viscosity: float = 0.05
    kind: str = "bgk"
    high_order_rate: float = 1.0
    policy: str = "constant"
    policy_eps0: float = 0.01
    explicit_rates: Optional[Sequence[float]] = None
    faces: List[FaceSpec] = field(default_factory=lambda: [FaceSpec() for _ in range(6)])
    body_force: Sequence[float] = (0.0, 0.0, 0.0)
    solids: List[SolidConfig] = field(default_factory=list)
    emitters: List[TracerEmitter] = field(default_factory=list)
    init: str = "uniform"
    init_density: float = 1.0
    init_velocity: Sequence[float] = (0.0, 0.0, 0.0)
    tg_u_max: float = 0.02
    steps: int = 0
    regions: int = 1
    threads_per_region: int = 0
    alpha: int = 1
    block_edge: int = 1
    ib_mode: str = "atomic"
    seed: int = 1

    @property
    def dims(self):
        return (self.nx, self.ny, self.nz)

    @property
    def n_nodes(self) -> int:
        return self.nx * self.ny * self.nz

    def to_c(self) -> "CScene":
        return CScene(self)


def _v3(dst, src):
    for a in range(3):
        dst[a] = float(src[a])


class CScene:
    """Owns the C struct (and its solids array) for the duration of a call."""

    def __init__(self, cfg: SceneConfig):
        c = _abi.SceneConfigC()
        try:
            c.nx, c.ny, c.nz = int(cfg.nx), int(cfg.ny), int(cfg.nz)
            c.viscosity = float(cfg.viscosity)
            c.kind = KINDS[cfg.kind]
            c.high_order_rate = float(cfg.high_order_rate)
            c.policy = POLICIES[cfg.policy]
            c.policy_eps0 = float(cfg.policy_eps0)
            if cfg.explicit_rates is not None:
                c.has_explicit_rates = 1
                for i in range(27):
                    c.rates[i] = float(cfg.explicit_rates[i])
            for f in range(6):
                c.faces[f].condition = CONDITIONS[cfg.faces[f].condition]
                _v3(c.faces[f].velocity, cfg.faces[f].velocity)
            _v3(c.body_force, cfg.body_force)
            self.solids = (_abi.SolidConfigC * max(1, len(cfg.solids)))()
            for k, s in enumerate(cfg.solids):
                sc = self.solids[k]
                m = s.mesh
                sc.mesh.type = MESHES[m.type]
                _v3(sc.mesh.center, m.center)
                _v3(sc.mesh.lo, m.lo)
                _v3(sc.mesh.hi, m.hi)
                _v3(sc.mesh.origin, m.origin)
                sc.mesh.radius = float(m.radius)
                sc.mesh.subdivisions = int(m.subdivisions)
                sc.mesh.fins = int(m.fins)
                sc.mesh.fin_length = float(m.fin_length)
                sc.mesh.fin_height = float(m.fin_height)
                sc.mesh.fin_spacing = float(m.fin_spacing)
                sc.mesh.size = float(m.size)
                sc.mesh.plane_z = float(m.plane_z)
                sc.poisson_radius = float(s.poisson_radius)
                sc.sampling = SAMPLING[s.sampling]
                if s.motion is not None:
                    sc.has_motion = 1
                    _v3(sc.linear_velocity, s.motion.linear_velocity)
                    _v3(sc.angular_velocity, s.motion.angular_velocity)
                    _v3(sc.center, s.motion.center)
            c.n_solids = len(cfg.solids)
            c.solids = C.cast(self.solids, C.POINTER(_abi.SolidConfigC))
            c.init = INITS[cfg.init]
            c.init_density = float(cfg.init_density)
            _v3(c.init_velocity, cfg.init_velocity)
            c.tg_u_max = float(cfg.tg_u_max)
            c.regions = int(cfg.regions)
            c.threads_per_region = int(cfg.threads_per_region)
            c.alpha = int(cfg.alpha)
            c.block_edge = int(cfg.block_edge)
            c.ib_mode = IB_MODES[cfg.ib_mode]
            c.seed = int(cfg.seed) & 0xFFFFFFFFFFFFFFFF
        except KeyError as e:
            raise ConfigError(f"config: unknown enum value {e}") from None
        self.c = c

    @property
    def ptr(self):
        return C.byref(self.c)


# ---- JSON schema (scene.cpp:132-331) ------------------------------------

def _fail(path, msg):
    raise ConfigError(f"config: {path}: {msg}")


def _check_keys(j, path, keys):
    if not isinstance(j, dict):
        _fail(path, "must be an object")
    for k in j:
        if k not in keys:
            _fail(f"{path}.{k}", "unknown key")


def _num(j, path):
    if isinstance(j, bool) or not isinstance(j, (int, float)):
        _fail(path, "must be a number")
    if not math.isfinite(j):
        _fail(path, "must be finite")
    return float(j)


def _vec3(j, path):
    if not isinstance(j, list) or len(j) != 3:
        _fail(path, "must be an array of 3 numbers")
    return tuple(_num(j[a], f"{path}[{a}]") for a in range(3))


def _int(j, path, lo, hi):
    if isinstance(j, bool) or not isinstance(j, int):
        _fail(path, "must be an integer")
    if j < lo or j > hi:
        _fail(path, f"must be in [{lo}, {hi}]")
    return int(j)


def _enum(j, path, table):
    if j not in table:
        _fail(path, "must be one of " + "|".join(table))
    return j


def _mesh(j, path) -> MeshConfig:
    t = j.get("type", "") if isinstance(j, dict) else ""
    m = MeshConfig(type=t)
    if t == "sphere":
        _check_keys(j, path, {"type", "center", "radius", "subdivisions"})
        m.center = _vec3(j["center"], path + ".center")
        m.radius = _num(j["radius"], path + ".radius")
        if m.radius <= 0:
            _fail(path + ".radius", "must be > 0")
        m.subdivisions = _int(j["subdivisions"], path + ".subdivisions", 0, 7) if "subdivisions" in j else 3
    elif t == "box":
        _check_keys(j, path, {"type", "lo", "hi"})
        m.lo = _vec3(j["lo"], path + ".lo")
        m.hi = _vec3(j["hi"], path + ".hi")
    elif t == "fin-comb":
        _check_keys(j, path, {"type", "origin", "fins", "fin_length", "fin_height", "fin_spacing"})
        m.origin = _vec3(j["origin"], path + ".origin")
        m.fins = _int(j["fins"], path + ".fins", 1, 4096)
        m.fin_length = _num(j["fin_length"], path + ".fin_length")
        m.fin_height = _num(j["fin_height"], path + ".fin_height")
        m.fin_spacing = _num(j["fin_spacing"], path + ".fin_spacing")
    elif t == "quad":
        _check_keys(j, path, {"type", "size", "z"})
        m.size = _num(j["size"], path + ".size")
        m.plane_z = _num(j["z"], path + ".z") if "z" in j else 0.0
    elif t == "file":
        _fail(path + ".type", "mesh files are host assets; load them with the reference tools")
    else:
        _fail(path + ".type", "must be one of sphere|box|fin-comb|quad|file")
    return m


def parse_scene_config(text: str) -> SceneConfig:
    """parse_scene_config (scene.cpp:132-331): strict keys, validated ranges."""
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise ConfigError(f"config: invalid JSON: {e}") from None
    _check_keys(j, "$", {"grid", "viscosity", "collision", "faces", "body_force", "solids", "tracers",
                          "initial", "steps", "output_cadence", "output_dir", "regions", "threads_per_region",
                          "layout", "ib_accumulation", "tune", "seed"})
    cfg = SceneConfig()
    grid = j["grid"]
    _check_keys(grid, "$.grid", {"nx", "ny", "nz"})
    cfg.nx = _int(grid["nx"], "$.grid.nx", 2, 4096)
    cfg.ny = _int(grid["ny"], "$.grid.ny", 2, 4096)
    cfg.nz = _int(grid["nz"], "$.grid.nz", 2, 4096)
    cfg.viscosity = _num(j["viscosity"], "$.viscosity")
    if not cfg.viscosity > 0:
        _fail("$.viscosity", "must be > 0")
    col = j["collision"]
    _check_keys(col, "$.collision", {"kind", "high_order_rate", "rates", "policy", "policy_eps0"})
    cfg.kind = _enum(col["kind"], "$.collision.kind", KINDS)
    if "high_order_rate" in col:
        cfg.high_order_rate = _num(col["high_order_rate"], "$.collision.high_order_rate")
    if "policy" in col:
        cfg.policy = _enum(col["policy"], "$.collision.policy", POLICIES)
    if "policy_eps0" in col:
        cfg.policy_eps0 = _num(col["policy_eps0"], "$.collision.policy_eps0")
        if cfg.policy_eps0 <= 0:
            _fail("$.collision.policy_eps0", "must be > 0")
    if "rates" in col:
        r = col["rates"]
        if not isinstance(r, list) or len(r) != 27:
            _fail("$.collision.rates", "must be an array of 27 numbers")
        cfg.explicit_rates = [_num(r[i], f"$.collision.rates[{i}]") for i in range(27)]
    faces = j["faces"]
    _check_keys(faces, "$.faces", set(FACE_NAMES))
    cfg.faces = []
    for name in FACE_NAMES:
        fp = f"$.faces.{name}"
        if name not in faces:
            _fail(fp, "missing face")
        fj = faces[name]
        _check_keys(fj, fp, {"condition", "velocity"})
        fs = FaceSpec(condition=_enum(fj["condition"], fp + ".condition", CONDITIONS))
        if "velocity" in fj:
            fs.velocity = _vec3(fj["velocity"], fp + ".velocity")
        cfg.faces.append(fs)
    for a in range(3):
        if (cfg.faces[2 * a].condition == "periodic") != (cfg.faces[2 * a + 1].condition == "periodic"):
            raise ConfigError(f"boundary: periodic faces must come in opposing pairs (axis {a})")
    if "body_force" in j:
        cfg.body_force = _vec3(j["body_force"], "$.body_force")
    for idx, sj in enumerate(j.get("solids", [])):
        sp = f"$.solids[{idx}]"
        _check_keys(sj, sp, {"mesh", "poisson_radius", "sampling", "motion"})
        sc = SolidConfig(mesh=_mesh(sj["mesh"], sp + ".mesh"))
        sc.poisson_radius = _num(sj["poisson_radius"], sp + ".poisson_radius")
        if sc.poisson_radius <= 0:
            _fail(sp + ".poisson_radius", "must be > 0")
        if "sampling" in sj:
            sc.sampling = _enum(sj["sampling"], sp + ".sampling", SAMPLING)
        if "motion" in sj:
            mj = sj["motion"]
            _check_keys(mj, sp + ".motion", {"linear_velocity", "angular_velocity", "center"})
            mo = RigidMotion()
            if "linear_velocity" in mj:
                mo.linear_velocity = _vec3(mj["linear_velocity"], sp + ".motion.linear_velocity")
            if "angular_velocity" in mj:
                mo.angular_velocity = _vec3(mj["angular_velocity"], sp + ".motion.angular_velocity")
            if "center" in mj:
                mo.center = _vec3(mj["center"], sp + ".motion.center")
            sc.motion = mo
        cfg.solids.append(sc)
    for idx, tj in enumerate(j.get("tracers", [])):  # scene.cpp:244-258
        tp = f"$.tracers[{idx}]"
        _check_keys(tj, tp, {"region", "rate"})
        rj = tj["region"]
        _check_keys(rj, tp + ".region", {"lo", "hi"})
        cfg.emitters.append(TracerEmitter(lo=_vec3(rj["lo"], tp + ".region.lo"),
                                          hi=_vec3(rj["hi"], tp + ".region.hi"),
                                          rate=_int(tj["rate"], tp + ".rate", 0, 1000000)))
    if "initial" in j:
        ij = j["initial"]
        t = ij.get("type", "uniform")
        if t == "uniform":
            _check_keys(ij, "$.initial", {"type", "density", "velocity"})
            if "density" in ij:
                cfg.init_density = _num(ij["density"], "$.initial.density")
                if cfg.init_density <= 0:
                    _fail("$.initial.density", "must be > 0")
            if "velocity" in ij:
                cfg.init_velocity = _vec3(ij["velocity"], "$.initial.velocity")
        elif t == "taylor-green":
            _check_keys(ij, "$.initial", {"type", "u_max"})
            cfg.init = "taylor-green"
            if "u_max" in ij:
                cfg.tg_u_max = _num(ij["u_max"], "$.initial.u_max")
        else:
            _fail("$.initial.type", "must be uniform|taylor-green")
    if "steps" in j:
        cfg.steps = _int(j["steps"], "$.steps", 0, 100000000)
    if "regions" in j:
        cfg.regions = _int(j["regions"], "$.regions", 1, 1024)
    if cfg.regions > cfg.nz:
        _fail("$.regions", "must be <= grid.nz")
    if "threads_per_region" in j:
        cfg.threads_per_region = _int(j["threads_per_region"], "$.threads_per_region", 0, 4096)
    if "layout" in j:
        lj = j["layout"]
        _check_keys(lj, "$.layout", {"alpha", "block_edge"})
        if "alpha" in lj:
            cfg.alpha = _int(lj["alpha"], "$.layout.alpha", 1, 1 << 30)
        if "block_edge" in lj:
            cfg.block_edge = _int(lj["block_edge"], "$.layout.block_edge", 1, 4096)
    if "ib_accumulation" in j:
        cfg.ib_mode = _enum(j["ib_accumulation"], "$.ib_accumulation", IB_MODES)
    if "seed" in j:
        cfg.seed = int(j["seed"])
    for f in range(6):
        if cfg.faces[f].condition == "outflow" and cfg.dims[f // 2] < 2:
            _fail("$.faces", "outflow requires extent >= 2 on its axis")
    return cfg


def load_scene_config(path: str) -> SceneConfig:
    try:
        with open(path) as fh:
            text = fh.read()
    except OSError:
        raise ConfigError(f"cannot open config file: {path}") from None
    return parse_scene_config(text)
