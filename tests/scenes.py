"""Parity scenes shared by the tests (SURVEY.md §8(d) configs and their
small twins).  All use cm-mrt + relax-toward-one with high_order_rate 1.5 so
the adaptive (ACM) path is exercised."""
from paper_2101_11856_b200 import FaceSpec, MeshConfig, RigidMotion, SceneConfig, SolidConfig


def acm(cfg: SceneConfig) -> SceneConfig:
    cfg.kind = "cm-mrt"
    cfg.high_order_rate = 1.5
    cfg.policy = "relax-toward-one"
    cfg.policy_eps0 = 0.01
    return cfg


def faces(*conds, inlet=(0.05, 0.0, 0.0)):
    out = []
    for c in conds:
        out.append(FaceSpec(c, inlet if c == "inlet" else (0.0, 0.0, 0.0)))
    return out


def cavity(n=64, nu=0.02, lid=0.05) -> SceneConfig:
    """C1: lid-driven cavity, z+ inlet lid, other faces no-slip."""
    cfg = acm(SceneConfig(nx=n, ny=n, nz=n, viscosity=nu))
    cfg.faces = faces("no-slip", "no-slip", "no-slip", "no-slip", "no-slip", "inlet", inlet=(lid, 0.0, 0.0))
    return cfg


def closed_box(n=16, u0=(0.02, -0.01, 0.005)) -> SceneConfig:
    cfg = acm(SceneConfig(nx=n, ny=n + 2, nz=n + 1, viscosity=0.02))
    cfg.init_velocity = u0
    return cfg


def taylor_green(nx=64, ny=64, nz=4, nu=0.02, kind="cm-mrt") -> SceneConfig:
    cfg = acm(SceneConfig(nx=nx, ny=ny, nz=nz, viscosity=nu))
    cfg.kind = kind
    cfg.faces = faces(*["periodic"] * 6)
    cfg.init = "taylor-green"
    cfg.tg_u_max = 0.02
    return cfg


def sphere(nx=256, ny=128, nz=128, center=(80, 64, 64), radius=16.0, subdiv=4, r=0.5) -> SceneConfig:
    """C2: flow past a sphere, x- inlet, x+ outflow, y/z no-slip."""
    cfg = acm(SceneConfig(nx=nx, ny=ny, nz=nz, viscosity=0.02))
    cfg.faces = faces("inlet", "outflow", "no-slip", "no-slip", "no-slip", "no-slip")
    cfg.init_velocity = (0.05, 0.0, 0.0)
    cfg.solids = [SolidConfig(MeshConfig(type="sphere", center=center, radius=radius, subdivisions=subdiv),
                              poisson_radius=r)]
    cfg.block_edge = 2
    cfg.seed = 1
    return cfg


def channel(n=128, nz=None) -> SceneConfig:
    """C3 twin: y walls, x and z periodic, body force along z."""
    cfg = acm(SceneConfig(nx=n, ny=n, nz=nz or n, viscosity=0.002))
    cfg.faces = faces("periodic", "periodic", "no-slip", "no-slip", "periodic", "periodic")
    cfg.body_force = (0.0, 0.0, 1e-6)
    return cfg


def rotating_fins(nx=128, ny=64, nz=64) -> SceneConfig:
    """C5 twin: rotating fin comb about x (SURVEY App. B `twins`)."""
    import math
    cfg = acm(SceneConfig(nx=nx, ny=ny, nz=nz, viscosity=0.02))
    cfg.faces = faces("no-slip", "no-slip", "no-slip", "no-slip", "no-slip", "no-slip")
    cfg.solids = [SolidConfig(MeshConfig(type="fin-comb", origin=(52, 22, 22), fins=8, fin_length=20,
                                         fin_height=16, fin_spacing=2.5), poisson_radius=0.5,
                              motion=RigidMotion(angular_velocity=(2 * math.pi / 500, 0, 0),
                                                 center=(62, 30.75, 30)))]
    cfg.block_edge = 2
    return cfg


def outflow_mix(nx=10, ny=8, nz=7) -> SceneConfig:
    """Edge semantics stress: outflow faces meeting no-slip/inlet/outflow
    (stale outflow-edge reads)."""
    cfg = acm(SceneConfig(nx=nx, ny=ny, nz=nz, viscosity=0.05))
    cfg.faces = faces("inlet", "outflow", "no-slip", "outflow", "outflow", "inlet", inlet=(0.03, 0.01, -0.01))
    cfg.init_velocity = (0.02, 0.0, 0.0)
    return cfg


def city(nx=64, ny=32, nz=48, n_boxes=4, seed=7, r=0.7) -> SceneConfig:
    """C4 twin: seeded synthetic "city" of box solids on a no-slip ground,
    x- inlet 0.05, x+ outflow (Poisson r=0.7, since r=0.5
    boxes diverge)."""
    import numpy as np
    cfg = acm(SceneConfig(nx=nx, ny=ny, nz=nz, viscosity=0.02))
    cfg.faces = faces("inlet", "outflow", "no-slip", "no-slip", "no-slip", "no-slip")
    cfg.init_velocity = (0.05, 0.0, 0.0)
    rng = np.random.default_rng(seed)
    cfg.solids = []
    for _ in range(n_boxes):
        w, d = rng.uniform(4, 8, size=2)
        h = rng.uniform(6, 0.6 * ny)
        x0 = rng.uniform(0.25 * nx, 0.75 * nx - w)
        z0 = rng.uniform(6, nz - 6 - d)
        cfg.solids.append(SolidConfig(MeshConfig(type="box", lo=(x0, 1.2, z0), hi=(x0 + w, 1.2 + h, z0 + d)),
                                      poisson_radius=r))
    cfg.block_edge = 2
    return cfg


def city_c4(n_boxes=220, seed=7, r=0.7, nx=1200, ny=250, nz=840) -> SceneConfig:
    """configs[3] at full size: 1200x250x840 "smoke through complex
    architecture" — a seeded city of box solids (Poisson r = 0.7), x- inlet,
    x+ outflow, no-slip ground and walls; ~3.5 M solid samples."""
    import numpy as np
    cfg = acm(SceneConfig(nx=nx, ny=ny, nz=nz, viscosity=0.02))
    cfg.faces = faces("inlet", "outflow", "no-slip", "no-slip", "no-slip", "no-slip")
    cfg.init_velocity = (0.05, 0.0, 0.0)
    rng = np.random.default_rng(seed)
    cfg.solids = []
    # non-overlapping lots (overlapping boxes double the local sample density,
    # which the unnormalised penalty force does not survive)
    lots = [(150 + 50 * i, 20 + 50 * k) for i in range((nx - 300) // 50) for k in range((nz - 40) // 50)]
    for j in rng.permutation(len(lots))[:n_boxes]:
        lx, lz = lots[j]
        w, d = rng.uniform(10, 40, size=2)
        h = rng.uniform(20, 200)
        x0 = lx + rng.uniform(0, 45 - w)
        z0 = lz + rng.uniform(0, 45 - d)
        cfg.solids.append(SolidConfig(MeshConfig(type="box", lo=(x0, 1.2, z0), hi=(x0 + w, 1.2 + h, z0 + d)),
                                      poisson_radius=r))
    cfg.block_edge = 2
    return cfg


def city_twin(seed=7, r=0.7) -> SceneConfig:
    """configs[3] 1/8-scale parity twin (SURVEY §8(d) C4 row, App. B `twins`
    (3)): 150x64x105, 12 seeded boxes with footprints 4..12, heights 8..40 on
    base y = 1.2, x in [30, 120], z in [8, 85]; Poisson r = 0.7."""
    import numpy as np
    cfg = acm(SceneConfig(nx=150, ny=64, nz=105, viscosity=0.02))
    cfg.faces = faces("inlet", "outflow", "no-slip", "no-slip", "no-slip", "no-slip")
    cfg.init_velocity = (0.05, 0.0, 0.0)
    rng = np.random.default_rng(seed)
    cfg.solids = []
    # 12 non-overlapping lots of 22 x 19 cells inside x [30, 120], z [8, 85]
    lots = [(30 + 22 * i, 8 + 19 * k) for i in range(4) for k in range(4)]
    for j in rng.permutation(len(lots))[:12]:
        lx, lz = lots[j]
        w, d = rng.uniform(4, 12, size=2)
        h = rng.uniform(8, 40)
        x0 = lx + rng.uniform(0, 20 - w)
        z0 = lz + rng.uniform(0, 17 - d)
        cfg.solids.append(SolidConfig(MeshConfig(type="box", lo=(x0, 1.2, z0), hi=(x0 + w, 1.2 + h, z0 + d)),
                                      poisson_radius=r))
    cfg.block_edge = 2
    return cfg


def fan_c5(r=0.5) -> SceneConfig:
    """configs[4] at full size: rotating fan (8-fin comb about x) in a closed
    512x256x256 box, one revolution per 2000 steps (tip speed ~0.25)."""
    import math
    cfg = acm(SceneConfig(nx=512, ny=256, nz=256, viscosity=0.02))
    cfg.faces = faces(*["no-slip"] * 6)
    cfg.solids = [SolidConfig(MeshConfig(type="fin-comb", origin=(208, 88, 88), fins=8, fin_length=80,
                                         fin_height=64, fin_spacing=10.0), poisson_radius=r,
                              motion=RigidMotion(angular_velocity=(2 * math.pi / 2000, 0, 0),
                                                 center=(248, 123, 120)))]
    cfg.block_edge = 2
    return cfg
