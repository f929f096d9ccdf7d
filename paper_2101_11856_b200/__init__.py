"""B200-native ACM-MRT + immersed-boundary lattice-Boltzmann step
(arXiv 2101.11856) behind the reference solver's API.

    from paper_2101_11856_b200 import SceneConfig, build_scene, Runner
    scene = build_scene(cfg)          # host setup (sampling, ordering)
    r = Runner(scene)                 # device state on cuda:0
    r.advance(100)                    # fused sm_100a step kernels
    rho = r.gather_rho()              # canonical AoS FP64 readback
"""
from .scene import (ConfigError, FaceSpec, MeshConfig, RigidMotion, SceneConfig, SolidConfig, TracerEmitter,
                    load_scene_config, parse_scene_config)
from .runner import (CudaError, Runner, Scene, StateError, StepStatus, TimingRow, build_scene,
                     collide_batch, device_count, dump_field, emit_tracers, lib, model_rates, morton3, rasterize_density,
                     reorder_permutation, split_domain, TracerCloud, ib_kernel_support, ib_interpolate_velocity,
                     ib_penalty_forces, ib_spread_forces, ib_update_rigid_motion, ib_reaction_totals)

from . import autotune
from .autotune import TuneOutcome, TuneSpec

__all__ = [
    "autotune", "TuneOutcome", "TuneSpec",
    "ConfigError", "FaceSpec", "MeshConfig", "RigidMotion", "SceneConfig", "SolidConfig",
    "load_scene_config", "parse_scene_config", "CudaError", "Runner", "Scene", "StateError",
    "StepStatus", "TimingRow", "build_scene", "collide_batch", "device_count", "dump_field", "lib", "model_rates",
    "morton3", "reorder_permutation", "split_domain", "TracerEmitter", "TracerCloud", "emit_tracers",
    "rasterize_density", "ib_kernel_support", "ib_interpolate_velocity", "ib_penalty_forces", "ib_spread_forces",
    "ib_update_rigid_motion", "ib_reaction_totals",
]
