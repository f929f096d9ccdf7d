#!/usr/bin/env python
"""Summarise ncu captures into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py <tag> <config>=<report.ncu-rep> ... [--launches <config>=<launches.csv> ...]

Writes profiles/ncu_<tag>.md (human summary: per-kernel time, DRAM bytes,
throughput, registers, occupancy, top stall reasons) and merges the
per-config numbers bench.py reads (dominant-kernel DRAM bytes per launch)
into profiles/ncu_summary.json.
"""
from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_pct"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_pct"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("launch__shared_mem_per_block_dynamic", "dyn_smem"),
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
              "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "s": 1, "second": 1}


def raw_rows(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def value(h, units, r, name):
    if name not in h:
        return None
    i = h.index(name)
    try:
        v = float(r[i].replace(",", ""))
    except ValueError:
        return r[i]
    return v * UNIT_SCALE.get(units[i], 1)


def stalls(h, r):
    pre = "smsp__pcsamp_warps_issue_stalled_"
    d = {}
    for i, w in enumerate(h):
        if w.startswith(pre) and not w.endswith("_not_issued"):
            try:
                d[w[len(pre):]] = float(r[i].replace(",", ""))
            except ValueError:
                pass
    tot = sum(d.values()) or 1.0
    return sorted(((k, v / tot) for k, v in d.items()), key=lambda kv: -kv[1])[:5]


def launches(csv_path: str):
    rows = list(csv.reader(open(csv_path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    return [(k, len(v), sum(v) / len(v), sum(v) / tot) for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))]


def main():
    tag = sys.argv[1]
    reps, lls = {}, {}
    mode = reps
    for a in sys.argv[2:]:
        if a == "--launches":
            mode = lls
            continue
        k, v = a.split("=", 1)
        mode[k] = v
    summ_path = ROOT / "profiles" / "ncu_summary.json"
    summ = json.loads(summ_path.read_text()) if summ_path.exists() else {}
    md = [f"# ncu summary `{tag}`", "",
          "Captured with `ncu --set full --clock-control none --import-source on` on one B200 "
          "(per-launch times are cold-cache, serialised replays: compare shares, not absolutes).", ""]
    for cfg, rep in reps.items():
        h, units, rows = raw_rows(rep)
        md += [f"## {cfg}: `{Path(rep).name}`", "",
               "| kernel | time us | DRAM rd MB | DRAM wr MB | DRAM % | regs | warps act % | issue % | FMA pipe % | top stalls |",
               "|---|---|---|---|---|---|---|---|---|---|"]
        best = None
        for r in rows:
            name = value(h, units, r, "Kernel Name") if "Kernel Name" in h else r[4]
            v = {key: value(h, units, r, m) for m, key in METRICS}
            st = ", ".join(f"{k} {p:.0%}" for k, p in stalls(h, r)[:3])
            short = str(name).split("(")[0].replace("void ", "")
            md.append(f"| `{short}` | {v['time'] * 1e6:.1f} | {v['dram_read'] / 1e6:.1f} | {v['dram_write'] / 1e6:.1f} | "
                      f"{v['dram_pct']:.1f} | {int(v['regs'])} | {v['warps_active_pct']:.1f} | {v['issue_pct']:.1f} | "
                      f"{v['fma_pipe_pct']:.1f} | {st} |")
            # the steady-state step: the launch with the least DRAM traffic (a
            # launch that also stores rho*/u* moves 16 B/node more)
            tr = v["dram_read"] + v["dram_write"]
            if ("fluid_bulk" in short or "fluid_ghost" in short) and (
                    best is None or tr < best["dram_read"] + best["dram_write"]):
                best = dict(v, kernel=short)
        md.append("")
        if best:
            summ[cfg] = {"tag": tag, "kernel": best["kernel"],
                         "fluid_dram_bytes_per_launch": best["dram_read"] + best["dram_write"],
                         "ncu_time_s": best["time"], "regs": best["regs"]}
    for cfg, path in lls.items():
        md += [f"## launch list {cfg}: `{Path(path).name}` (`--metrics gpu__time_duration.sum`)", "",
               "| kernel | launches | avg us | share |", "|---|---|---|---|"]
        for k, n, avg, share in launches(path):
            md.append(f"| `{k.replace('void ', '')}` | {n} | {avg / 1e3:.1f} | {share:.1%} |")
        md.append("")
    (ROOT / "profiles").mkdir(exist_ok=True)
    (ROOT / "profiles" / f"ncu_{tag}.md").write_text("\n".join(md) + "\n")
    summ_path.write_text(json.dumps(summ, indent=1) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
