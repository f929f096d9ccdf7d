#!/usr/bin/env python
"""Eq. 10 sweep on the device (the `lbm tune` verb's GPU counterpart): prints
the cost surface (Fig. 9 analog) and the chosen (variant, ell, alpha) as JSON.

    python tools/tune.py [--config c2|c3|c1] [--steps 10] [--warmup 5] [--ell-max L] [--alphas 256,4096,...]
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_2101_11856_b200 as lbm  # noqa: E402
from paper_2101_11856_b200 import autotune  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2", choices=sorted(bench.CONFIGS))
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--ell-max", type=int, default=None)
    ap.add_argument("--alphas", default=None)
    ap.add_argument("--variants", default="0:0,0:1,1:0,1:1",
                    help="fluid:ib[:cta] list; cta = staged-kernel threads per CTA (512/256/128)")
    a = ap.parse_args()
    cfg, desc = bench.CONFIGS[a.config](1)
    scene = lbm.build_scene(cfg)
    variants = [tuple(int(x) for x in v.split(":")) for v in a.variants.split(",")]
    spec = autotune.TuneSpec.from_scene(scene, n_steps=a.steps, warmup=a.warmup, variants=variants)
    if a.ell_max:
        spec.ell_max = min(spec.ell_max, a.ell_max)
    if a.alphas:
        spec.alphas = [int(x) for x in a.alphas.split(",")]
    base = lbm.Runner(scene)
    out = autotune.search(base, spec)
    print(json.dumps({"workload": desc, "candidates": spec.candidate_count(),
                      "chosen": {"variant": out.variant, "ell": out.ell, "alpha": out.alpha,
                                 "ms_per_step": out.cost * 1e3},
                      "rows": [[r.variant, r.ell, r.alpha, r.seconds * 1e3] for r in out.rows]}))


if __name__ == "__main__":
    main()
