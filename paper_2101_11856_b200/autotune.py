"""Parametric cost model and exhaustive search (paper Eq. 10, SPEC [MODULE]
autotune), the GPU counterpart of /root/reference/proj/src/autotune.cpp.

Semantics kept from the reference:
  * TuneSpec.from_scene (autotune.cpp:9-27): ell in {1..L_m}, L_m = the
    solids' smallest bbox edge (1 without solids); alpha in {2^1..2^floor(log2 N)}.
  * measure_cost (autotune.cpp:29-36): set_layout, warm-up, mean seconds per
    step over n_steps, +inf on divergence — timed on the device with CUDA
    events (Runner.measure_cost).
  * search_with_cost (autotune.cpp:38-60): argmin over the full grid, ties
    toward smaller ell then smaller alpha (ascending enumeration, strict <);
    raises ConfigError if every candidate is invalid; full cost table kept.
  * search (autotune.cpp:62-70): runs on a clone; the probe keeps advancing.

B200 extensions:
  * the kernel variant is a third, outermost search dimension (the paper's
    "launch split chosen from the cost model"; the reference fixes the
    two-pass split at kSplitBoundary = 14, collision.hpp:58): fluid kernel
    (TMA-staged ghost layout / register-direct compact layout) x IB pipeline
    (fused / split), ties toward variant (0, 0); a variant may carry a third
    entry, the staged kernel's CTA shape (512 / 256 / 128 threads per CTA =
    1024 / 512 / 256-slot tiles, 0 = default) — the CTA-shape dimension;
  * alphas that map to the same device layout (Runner.layout_key) are
    measured once and share the cost, so a sweep is seconds, not minutes.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence, Tuple

from .scene import ConfigError


@dataclass
class TuneSpec:
    ell_min: int = 1
    ell_max: int = 1
    alphas: List[int] = field(default_factory=list)
    n_steps: int = 10
    warmup: int = 5
    variants: List[Tuple[int, ...]] = field(default_factory=lambda: [(0, 0)])

    def candidate_count(self) -> int:
        return (self.ell_max - self.ell_min + 1) * len(self.alphas) * len(self.variants)

    @staticmethod
    def from_scene(scene, n_steps: int = 10, warmup: int = 5,
                   variants: Optional[Sequence[Tuple[int, int]]] = None) -> "TuneSpec":
        """autotune.cpp:9-27."""
        cfg = scene.cfg
        spec = TuneSpec(n_steps=n_steps, warmup=warmup)
        if cfg.solids:
            min_edge = 1e300
            for s in range(len(cfg.solids)):
                smp = scene.samples(s)
                lo, hi = smp["bbox_lo"], smp["bbox_hi"]
                for a in range(3):
                    min_edge = min(min_edge, hi[a] - lo[a])
            spec.ell_max = max(1, int(math.floor(min_edge)))
        n = cfg.nx * cfg.ny * cfg.nz
        a = 2
        while a <= n:
            spec.alphas.append(a)
            a *= 2
        if not spec.alphas:
            spec.alphas.append(1)
        if spec.n_steps < 1:
            raise ConfigError("tune: n_steps must be >= 1")
        if variants is not None:
            spec.variants = list(variants)
        return spec


@dataclass
class TuneRow:
    ell: int
    alpha: int
    seconds: float
    variant: Tuple[int, ...] = (0, 0)


@dataclass
class TuneOutcome:
    ell: int = 0
    alpha: int = 0
    cost: float = math.inf
    variant: Tuple[int, ...] = (0, 0)
    rows: List[TuneRow] = field(default_factory=list)


def search_with_cost(spec: TuneSpec, cost: Callable[..., float]) -> TuneOutcome:
    """Pure argmin over the candidate grid (autotune.cpp:38-60).  `cost` takes
    (ell, alpha) or, with several variants, (ell, alpha, variant)."""
    out = TuneOutcome()
    with_variant = len(spec.variants) > 1 or spec.variants != [(0, 0)]
    for v in spec.variants:
        for ell in range(spec.ell_min, spec.ell_max + 1):
            for alpha in spec.alphas:
                c = cost(ell, alpha, v) if with_variant else cost(ell, alpha)
                out.rows.append(TuneRow(ell, alpha, c, v))
                if c < out.cost:  # strict: ties keep the earlier (smaller) candidate
                    out.cost, out.ell, out.alpha, out.variant = c, ell, alpha, v
    if not math.isfinite(out.cost):
        raise ConfigError("tune: every candidate was invalid")
    return out


def measure_cost(runner, ell: int, alpha: int, spec: TuneSpec) -> float:
    """autotune.cpp:29-36 on the device (the runner advances)."""
    return runner.measure_cost(ell, alpha, spec.warmup, spec.n_steps)


def _norm_variant(v) -> Tuple[int, int, int]:
    """(fluid, ib[, cta]) -> (fluid, ib, cta); cta 0 = the default shape."""
    v = tuple(int(x) for x in v)
    return (v + (0, 0, 0)[len(v):])[:3]


def _effective_cta(layout_key: int, cta: int) -> int:
    """CTA size the staged fluid launcher actually runs for a layout (a tile of
    2*cta slots must fit one Eq. 9 block; fluid.cu launch_ghost_planes)."""
    if not (layout_key >> 40) & 1:  # compact layout: no staged kernel
        return 0
    la = (layout_key >> 32) & 0xFF
    block = 1 << 62 if la == 31 else 1 << la
    want = cta or 512
    for t in (512, 256, 128):
        if t <= want and block >= 2 * t:
            return t
    return 128


def search(base, spec: TuneSpec, dedup: bool = True) -> TuneOutcome:
    """autotune.cpp:62-70: sweep on a clone of `base` (never alters its physics).

    Every variant is normalised to (fluid, ib, cta) and applied in full before
    a measurement, so a 2-entry variant never inherits the CTA shape of the
    previous one.  A CTA shape the launcher cannot honour for a layout (its
    tile would straddle an Eq. 9 block) is an invalid candidate (+inf), and
    the dedup key holds the shape that actually runs."""
    probe = base.clone()
    seen = {}

    def cost(ell, alpha, v=(0, 0)):
        nv = _norm_variant(v)
        if (tuple(probe.variant()) + (probe.cta(),)) != nv:
            probe.set_variant(nv[0], nv[1])
            probe.set_cta(nv[2])
        lkey = probe.layout_key(alpha)
        eff = _effective_cta(lkey, nv[2])
        if nv[2] and eff and eff != nv[2]:
            return math.inf
        key = (nv[0], nv[1], eff, ell, lkey) if dedup else None
        if key is not None and key in seen:
            return seen[key]
        c = measure_cost(probe, ell, alpha, spec)
        if key is not None:
            seen[key] = c
        return c

    return search_with_cost(spec, cost)


def apply(runner, outcome: TuneOutcome):
    """Apply a search result to the production runner (variant, CTA shape, layout)."""
    nv = _norm_variant(outcome.variant)
    runner.set_variant(nv[0], nv[1])
    runner.set_cta(nv[2])
    runner.set_layout(outcome.ell, outcome.alpha)
