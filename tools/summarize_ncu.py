"""Summarise ncu captures into profiles/ (run here, on the CPU box).

    python tools/summarize_ncu.py --rep gpurun_out/prof_r1.ncu-rep \
        --launches gpurun_out/launches.csv --tag r1_c2 --config c2

Writes profiles/<tag>_summary.md (per-kernel key metrics from the full
capture, the launch list aggregated per kernel with its share of device time,
top stall reasons of the MART kernel) and profiles/traffic.json (DRAM bytes per
launch of the MART kernel, read by bench.py as roofline.traffic).
"""
from __future__ import annotations

import argparse
import collections
import csv
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 pipe % of peak"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def ncu_csv(rep: str, page: str, kernel: str | None = None) -> list[list[str]]:
    cmd = ["ncu", "-i", rep, "--page", page, "--csv"]
    if kernel:
        cmd += ["--kernel-name", f"regex:{kernel}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


def to_bytes(v: str, unit: str) -> float:
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(v) * scale.get(unit, 1)


def launches(path: str):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ix = {k: i for i, k in enumerate(h)}
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) != len(h) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "")
        v = float(r[ix["Metric Value"]])
        u = r[ix["Metric Unit"]]
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(u, 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    return agg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--kernel", default="mart_wave_kernel")
    args = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)

    raw = ncu_csv(args.rep, "raw")
    h, units = raw[0], raw[1]
    ix = {k: i for i, k in enumerate(h)}
    lines = [f"# ncu summary `{args.tag}`", "", f"Source: `{os.path.basename(args.rep)}` "
             f"(`ncu --set full --clock-control none --import-source on`), config `{args.config}`.", "",
             "## Full capture, key metrics per profiled launch", "",
             "| kernel | " + " | ".join(n for _, n in KEYS) + " |",
             "|---|" + "---|" * len(KEYS)]
    traffic = None
    for r in raw[2:]:
        name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "")
        cells = []
        for k, _ in KEYS:
            if k in ix:
                cells.append(f"{r[ix[k]]} {units[ix[k]]}".strip())
            else:
                cells.append("-")
        lines.append(f"| `{name}` | " + " | ".join(cells) + " |")
        if args.kernel in name and traffic is None:
            rd = to_bytes(r[ix["dram__bytes_read.sum"]], units[ix["dram__bytes_read.sum"]])
            wr = to_bytes(r[ix["dram__bytes_write.sum"]], units[ix["dram__bytes_write.sum"]])
            dur = r[ix["gpu__time_duration.sum"]] + " " + units[ix["gpu__time_duration.sum"]]
            traffic = {"config": args.config, "kernel": name, "dram_bytes_per_launch": rd + wr,
                       "dram_read": rd, "dram_write": wr, "duration": dur, "source": os.path.basename(args.rep)}
    if args.launches:
        agg = launches(args.launches)
        tot = sum(v[1] for v in agg.values())
        lines += ["", "## Launch list (`--metrics gpu__time_duration.sum`, cold-cache, serialised)", "",
                  "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            lines.append(f"| `{k}` | {n} | {t / 1e3:.3f} | {100 * t / tot:.1f}% |")
    # stall reasons of the MART kernel
    src = ncu_csv(args.rep, "source", args.kernel)
    try:
        hh = src[1]
        sx = {k: i for i, k in enumerate(hh)}
        data = [r for r in src[2:] if len(r) == len(hh) and r[0] != "Address"]

        def num(x):
            try:
                return int(x)
            except ValueError:
                return 0
        tot = sum(num(r[sx["Warp Stall Sampling (All Samples)"]]) for r in data)
        stalls = [k for k in hh if k.startswith("stall_") and "Not Issued" not in k]
        agg = {k: sum(num(r[sx[k]]) for r in data) for k in stalls}
        lines += ["", f"## Warp stall reasons (first kernel of the source page: `{src[0][1][:60]}`)", "",
                  "| reason | share of samples |", "|---|---|"]
        for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]:
            lines.append(f"| {k} | {100 * v / max(tot, 1):.1f}% |")
    except Exception as e:  # the source page is optional
        lines += ["", f"(source page unavailable: {e})"]
    with open(os.path.join(PROF, f"{args.tag}_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if traffic:
        # one entry per configuration; the profile driver runs one MART
        # launch of one iteration, so a launch's DRAM bytes are an iteration's
        path = os.path.join(PROF, "traffic.json")
        try:
            with open(path) as f:
                allt = json.load(f)
            if "config" in allt:  # the round-1 single-entry layout
                allt = {}
        except Exception:
            allt = {}
        traffic["dram_bytes_per_iteration"] = traffic["dram_bytes_per_launch"]
        allt[args.config] = traffic
        with open(path, "w") as f:
            json.dump(allt, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
