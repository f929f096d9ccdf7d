#!/usr/bin/env python
"""Benchmark of the B200 ACM-MRT + IB lattice-Boltzmann step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c1|c3|c4|c5]

A "step" is one full time step (ghost fill = the six face passes, the IB
pass, the fused stream/moments/CM-MRT collision/forcing kernel) of the
workload.  Default: configs[1] of BASELINE.json (flow past a sphere
256x128x128 with 8,329 IB samples) on one GPU.  c1/c3/c4/c5 are configs[0],
[2], [3] and [4] at their named sizes.  N>1 (torchrun, one process per GPU):
c1/c2/c3 stack the per-GPU workload along z (weak scaling), c4/c5 split the
named domain (strong scaling); z-slab halos over NCCL.  Rank 0 prints one
JSON line.

--impl reference times the reference's own CPU implementation (the
unmodified reference compiled into oracle/_ref) on this box's host cores,
with the same `config` object.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

ALG_BYTES_PER_LU = 216          # 27 fp32 reads + 27 fp32 writes
IB_BYTES_PER_BAND_NODE = 68
IB_BYTES_PER_SAMPLE = 60


def c2_config(n_gpus: int):
    from tests import scenes
    import paper_2101_11856_b200 as lbm
    cfg = scenes.sphere()  # 256x128x128, sphere r=16 at (80,64,64), Poisson 0.5, seed 1, ell 2
    cfg.alpha = 1 << 22     # SoA on the device (set_layout is a pure permutation)
    if n_gpus > 1:          # weak scaling: one sphere per 128-plane slab
        cfg.nz = 128 * n_gpus
        cfg.solids = [lbm.SolidConfig(lbm.MeshConfig(type="sphere", center=(80, 64, 64 + 128 * k), radius=16.0,
                                                     subdivisions=4), poisson_radius=0.5) for k in range(n_gpus)]
    return cfg, "flow past a sphere 256x128x128 per GPU, D3Q27 ACM-MRT + IB (configs[1])", "weak"


def c3_config(n_gpus: int):
    from tests import scenes
    cfg = scenes.channel(n=512, nz=512 * n_gpus)
    cfg.alpha = 1 << 30
    return cfg, "channel 512^3 per GPU, D3Q27 ACM-MRT, z-periodic ring (configs[2])", "weak"


def c1_config(n_gpus: int):
    from tests import scenes
    cfg = scenes.cavity(n=64)
    cfg.alpha = 1 << 20
    return cfg, "lid-driven cavity 64^3 D3Q27 ACM-MRT (configs[0], L2-resident)", "weak"


def c4_config(n_gpus: int):
    from tests import scenes
    cfg = scenes.city_c4()
    cfg.alpha = 1 << 30
    return cfg, ("smoke through complex architecture 1200x250x840, 220 box solids, ~3.5M IB samples, "
                 "D3Q27 ACM-MRT + IB (configs[3], whole domain split over the GPUs)"), "strong"


def c5_config(n_gpus: int):
    from tests import scenes
    cfg = scenes.fan_c5()
    cfg.alpha = 1 << 30
    return cfg, "rotating fan 512x256x256, moving IB samples, D3Q27 ACM-MRT + IB (configs[4])", "strong"


CONFIGS = {"c2": c2_config, "c3": c3_config, "c1": c1_config, "c4": c4_config, "c5": c5_config}


def cpu_sample_config(cfg):
    """The CPU leg's bounded sample of a workload: the whole grid when its FP64
    reference state (488 B/node) fits comfortably in host memory, else a
    z-slab of it (the solids that intersect the slab are kept).  The reference
    runs its default layout (alpha = 1): the GPU arm's alpha is a device-layout
    hint, and the reference pads every field to a multiple of alpha (a 2^30
    alpha would allocate ~230 GB per field; results are layout-invariant)."""
    import copy
    n = cfg.nx * cfg.ny * cfg.nz
    max_nodes = 40_000_000  # ~20 GB of FP64 reference state
    sub = copy.deepcopy(cfg)
    sub.alpha = 1
    if n <= max_nodes:
        return sub, f"the full {cfg.nx}x{cfg.ny}x{cfg.nz} grid"
    nz = max(8, max_nodes // (cfg.nx * cfg.ny))
    sub.nz = nz
    keep = []
    for s in sub.solids:
        m = s.mesh
        zlo = m.lo[2] if m.type == "box" else (m.center[2] - m.radius if m.type == "sphere" else m.origin[2])
        if zlo + 2 < nz:
            if m.type == "box" and m.hi[2] > nz - 2:
                m.hi = (m.hi[0], m.hi[1], float(nz - 2))
            keep.append(s)
    sub.solids = keep
    return sub, f"a {cfg.nx}x{cfg.ny}x{nz} z-slab of the {cfg.nx}x{cfg.ny}x{cfg.nz} grid ({len(keep)} solids)"


def config_dict(cfg, desc, world, n_samples):
    """The `config` object, identical in both arms."""
    nodes = cfg.nx * cfg.ny * cfg.nz
    return {"workload": desc, "nodes": nodes, "nodes_per_gpu": nodes // world, "solid_samples": n_samples,
            "parallelism": f"z-slab x{world}", "layout": "SoA fp32 DDF-shifted (alpha >= n)",
            "l2": "inputs larger than L2 (f: %.2f GB/GPU vs 126 MB L2)" % (2 * 27 * 4 * nodes / world / 1e9)}


def scene_samples(cfg):
    import paper_2101_11856_b200 as lbm
    scene = lbm.build_scene(cfg)
    return scene, sum(len(scene.samples(s)["source_id"]) for s in range(len(cfg.solids)))


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML every
    ~2 ms (so even a 40 ms region yields a median), nvidia-smi as fallback."""

    # clocks_event_reasons bits (nvml.h)
    REASONS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
               "hw_thermal_slowdown": 0x40}

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, reason bits)
        self._stop = threading.Event()
        self._t = None
        self._ready = threading.Event()  # set once the first sample is in
        self.source = "nvml"

    def _run_nvml(self, nv):
        h = nv.nvmlDeviceGetHandleByIndex(self.index)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self._stop.is_set():
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            try:
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            except Exception:
                bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            self.samples.append((float(sm), float(mx), int(bits)))
            self._ready.set()
            self._stop.wait(0.002)

    def _run_smi(self):
        fields = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.active"]
        cmd = ["nvidia-smi", f"--id={self.index}", "--query-gpu=" + ",".join(fields), "--format=csv,noheader,nounits"]
        while not self._stop.is_set():
            try:
                out = subprocess.run(cmd, capture_output=True, text=True, timeout=5).stdout.strip().split(",")
                self.samples.append((float(out[0]), float(out[1]), int(out[2].strip(), 16)))
            except Exception:
                pass
            self._ready.set()
            self._stop.wait(0.05)

    def _run(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            try:
                self._run_nvml(nv)
            finally:
                nv.nvmlShutdown()
        except Exception:
            self.source = "nvidia-smi"
            self._run_smi()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        # NVML init can take longer than a short timed region: wait for the
        # first sample, then drop it, so every kept sample falls inside
        self._ready.wait(timeout=10.0)
        self.samples.clear()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"], "samples": 0}
        sm = [s[0] for s in self.samples]
        reasons = sorted({name for s in self.samples for name, bit in self.REASONS.items() if s[2] & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(s[1] for s in self.samples),
                "sm_mhz_min": min(sm), "reasons": reasons, "samples": len(self.samples), "source": self.source}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_traffic(config: str):
    """dram bytes per launch of the fluid kernel from the committed ncu summary."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    return d.get(config, {}).get("fluid_dram_bytes_per_launch")


def _time_reference(cfg, threads, warmup, runs, budget_s):
    """the reference Runner on `threads` host threads, `warmup`
    steps, then `runs` timed advance(k) calls (k sized to the budget); returns
    (median MLUPS, k, per-run seconds)."""
    from oracle.refpy import RefRunner
    r = RefRunner(cfg, threads=threads)
    t0 = time.perf_counter()
    r.advance(max(1, warmup))
    per = max((time.perf_counter() - t0) / max(1, warmup), 1e-4)
    k = max(1, min(50, int(budget_s / runs / per)))
    n = cfg.nx * cfg.ny * cfg.nz
    secs = []
    for _ in range(runs):
        t0 = time.perf_counter()
        r.advance(k)
        secs.append(time.perf_counter() - t0)
    return n * k / statistics.median(secs) / 1e6, k, secs


def cpu_baseline_sample(cfg, seconds: float = 15.0):
    """The reference (oracle/_ref) on this box's host cores: median of 5
    advance(k) runs after 2 warm-up steps, on a bounded sample of the workload."""
    threads = os.cpu_count() or 1
    sub, what = cpu_sample_config(cfg)
    v, k, secs = _time_reference(sub, threads, 2, 5, seconds)
    return {"value": v, "unit": "MLUPS", "cores": threads, "kind": "reference",
            "sample": f"median of 5 x advance({k}) after 2 warm-up steps on {what} "
                      f"(unmodified FP64 reference, {threads} threads; run seconds "
                      + ", ".join(f"{x:.2f}" for x in secs) + ")"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg, desc, scaling = CONFIGS[args.config](args.gpus)
    _, n_samples = scene_samples(cfg)
    threads = os.cpu_count() or 1
    sub, what = cpu_sample_config(cfg)
    from oracle.refpy import RefRunner
    r = RefRunner(sub, threads=threads)
    n = sub.nx * sub.ny * sub.nz
    w = max(2, args.warmup)
    t0 = time.perf_counter()
    r.advance(1)
    per = max(time.perf_counter() - t0, 1e-3)
    budget = 150.0
    w = max(1, min(w - 1, int(0.2 * budget / per)))
    k = max(1, min(args.steps, int(0.8 * budget / per)))
    r.advance(w)
    secs = []
    for _ in range(k):  # one timed advance(1) per step: the median is robust to host noise
        t0 = time.perf_counter()
        r.advance(1)
        secs.append(time.perf_counter() - t0)
    dt = sum(secs)
    v = n * k / dt / 1e6
    line = {
        "impl": "reference", "metric": "MLUPS (lattice-node updates/s, whole job)", "value": v, "unit": "MLUPS",
        "n_gpus": args.gpus, "steps": k, "warmup": w + 1, "ms_per_step": dt / k * 1e3, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(cfg, desc, args.gpus, n_samples),
        "cpu_baseline": {"value": v, "unit": "MLUPS", "cores": threads, "kind": "reference",
                         "sample": f"{k} timed steps (advance(1) each) on {what} after {w + 1} warm-up steps; "
                                   f"median step {statistics.median(secs) * 1e3:.1f} ms",
                         "median_mlups": n / statistics.median(secs) / 1e6},
        "e2e": {"value": v, "unit": "MLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import numpy as np
    import torch
    import paper_2101_11856_b200 as lbm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", device_id=device)
        dist = tdist
    if lbm.device_count() < 1:
        raise SystemExit("no CUDA device visible to the engine")

    cfg, desc, scaling = CONFIGS[args.config](world)
    scene, n_samples = scene_samples(cfg)
    # a dedicated (capturable) stream: the engine launches on it, the CUDA
    # events and NCCL synchronise with it
    stream = torch.cuda.Stream(device)
    torch.cuda.set_stream(stream)

    if world == 1:
        runner = lbm.Runner(scene, regions=1, device=local)
        runner.set_stream(stream.cuda_stream)
        stepper = None
    else:
        from paper_2101_11856_b200.dist import RankStepper
        runner = lbm.Runner(scene, device=local, world=world, rank=rank)
        dist.barrier()
        stepper = RankStepper(runner, dist, world, rank, cfg.faces[4].condition == "periodic", device)
    z0, z1 = runner.slab()
    nodes_local = cfg.nx * cfg.ny * (z1 - z0)
    nodes_global = cfg.nx * cfg.ny * cfg.nz

    def steps(k, macro_last=False):
        if stepper is None:
            st = runner.advance(k)
            if not st.ok:
                raise RuntimeError(f"diverged: {st}")
        else:
            for j in range(k):
                stepper.step(write_macro=macro_last and j == k - 1)

    # warm-up (also captures the CUDA graph)
    steps(max(3, args.warmup))
    if stepper is not None:
        stepper.finish()
    torch.cuda.synchronize(device)

    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        if dist:
            dist.barrier()
        torch.cuda.synchronize(device)
        start.record(stream)
        steps(args.steps)
        if stepper is not None:
            for w in stepper.pending:
                w.wait()
            stepper.pending = []
        end.record(stream)
        torch.cuda.synchronize(device)
        if dist:
            dist.barrier()
    ms = start.elapsed_time(end)
    if stepper is not None:
        st = stepper.finish()
        if not st.ok:
            raise RuntimeError(f"diverged: {st}")
    if dist:
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = nodes_global * args.steps / (ms * 1e-3) / 1e6

    # per-phase CUDA-event timing of the same step (fluid kernel share, roofline)
    rows = []
    kernels_per_step = runner.kernels_per_step() if stepper is None else None
    if stepper is None:
        runner.advance(min(args.steps, 20), timings=rows)
    fluid = [r.seconds for r in rows if r.phase == "fluid"]
    ib = [r.seconds for r in rows if r.phase == "ib"]
    bnd = [r.seconds for r in rows if r.phase == "boundary"]
    fluid_s = statistics.mean(fluid) if fluid else None
    peak, peak_kind = measured_peaks()
    roofline = None
    if fluid_s:
        alg = ALG_BYTES_PER_LU * nodes_local
        achieved = alg / fluid_s / 1e9
        traffic = ncu_traffic(args.config)
        step_bytes = alg + IB_BYTES_PER_SAMPLE * n_samples
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": traffic,
                    "kernel": "fluid_ghost_kernel (TMA-staged pull-stream + moments + CM-MRT/ACM + forcing)",
                    "alg_bytes_per_launch": alg, "alg_bytes_per_lu": ALG_BYTES_PER_LU,
                    "kernel_ms": fluid_s * 1e3, "peak_kind": peak_kind,
                    "boundary_ms": (statistics.mean(bnd) * 1e3) if bnd else 0.0,
                    "ib_ms": (statistics.mean(ib) * 1e3) if ib else 0.0,
                    "step_share_fluid": fluid_s / (ms_per_step * 1e-3),
                    "step_frac": step_bytes / (ms_per_step * 1e-3) / 1e9 / peak}

    # end-to-end through the public API: per step one advance(1) call with its
    # host inputs (motion-table rows) and host result (status + reaction totals)
    e2e = None
    if stepper is None:
        k_e2e = max(3, min(args.steps, 50))
        torch.cuda.synchronize(device)
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            st = runner.advance(1)
        rho_probe = None
        dt = time.perf_counter() - t0
        ns = len(cfg.solids)
        moving = sum(1 for s in cfg.solids if s.motion is not None)
        # runner.cpp advance(): the chunk start (8 B) + the motion rows of moving
        # solids up (static ones are uploaded once); counters (64 B, a 256 B slot
        # when solids are present) + the step's reaction totals down, one copy
        e2e = {"value": nodes_global * k_e2e / dt / 1e6, "unit": "MLUPS",
               "h2d_bytes_per_step": 8 + (2 * ns * 18 * 8 if moving else 0),
               "d2h_bytes_per_step": (256 + ns * 6 * 8) if ns else 64,
               "how": "one Runner.advance(1) call per step through the C ABI, host wall clock: each call "
                      "uploads that step's inputs (chunk start, motion rows of moving solids) from pinned host "
                      "memory and downloads its results (step counters/status + reaction totals) in one copy, "
                      "one stream sync",
               "steps": k_e2e}
        del rho_probe, st

    line = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline_sample(cfg)
        gpu_launches = kernels_per_step * args.steps if kernels_per_step else None
        line = {
            "metric": "MLUPS (lattice-node updates/s, whole job)", "value": value, "unit": "MLUPS",
            "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": config_dict(cfg, desc, world, n_samples),
            "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu,
            "clocks": clocks.summary(), "gpu_launches": gpu_launches,
            "per_gpu_mlups": value / world,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
