"""Summarise an ncu report (--set full) or a launch-list CSV into profiles/.

    python scripts/ncu_summary.py report.ncu-rep NAME [--config c4 --algo-bytes B]
    python scripts/ncu_summary.py launches.csv NAME --launches

Writes profiles/NAME.md (human-readable) and, with --config, merges the kernel's DRAM
traffic per launch into profiles/ncu_traffic.json (read by bench.py's roofline.traffic).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes_read.sum.per_second", "DRAM read BW"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed.sum", "warp instructions (SM)"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "fmaheavy pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def raw(rep: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {h: (v, u) for h, v, u in zip(hdr, r, units)}
        res.append(d)
    return res


def fnum(v: str) -> float:
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return float("nan")


def to_bytes(v: str, unit: str) -> float:
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return fnum(v) * scale


def summarise_report(rep: str, name: str, config: str | None, algo_bytes: float | None) -> None:
    rows = raw(rep)
    lines = [f"# {name}", "", f"source: `{os.path.basename(rep)}` (ncu --set full --clock-control none)", ""]
    traffic = []
    for d in rows:
        kname = d.get("Kernel Name", ("?", ""))[0]
        lines += [f"## {kname[:120]}", "", "| metric | value | unit |", "|---|---|---|"]
        for key, label in KEYS:
            if key in d:
                lines.append(f"| {label} (`{key}`) | {d[key][0]} | {d[key][1]} |")
        stalls = sorted(((k, fnum(v[0])) for k, v in d.items()
                         if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")),
                        key=lambda x: -x[1])[:8]
        if stalls:
            lines += ["", "top stall reasons (warps per issue-active cycle):", ""]
            lines += [f"- {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}: {v:.3f}"
                      for k, v in stalls]
        rd = to_bytes(*d["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in d else float("nan")
        wr = to_bytes(*d["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in d else float("nan")
        traffic.append(rd + wr)
        if algo_bytes:
            lines += ["", f"algorithmic bytes per launch: {algo_bytes:.6g}; DRAM traffic / algorithmic = "
                          f"{(rd + wr) / algo_bytes:.4f}"]
        lines.append("")
    os.makedirs(PROF, exist_ok=True)
    with open(os.path.join(PROF, f"{name}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if config and traffic:
        p = os.path.join(PROF, "ncu_traffic.json")
        db = json.load(open(p)) if os.path.exists(p) else {}
        db[config] = {"dram_bytes_per_launch": traffic[0], "report": name, "algorithmic_bytes": algo_bytes}
        with open(p, "w") as f:
            json.dump(db, f, indent=1, sort_keys=True)


def summarise_launches(path: str, name: str) -> None:
    txt = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.DictReader(txt))
    agg = defaultdict(list)
    for r in rows:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            agg[r["Kernel Name"]].append(fnum(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else
                                                                     (1.0 if r["Metric Unit"] == "us" else 1e3)))
    total = sum(sum(v) for v in agg.values())
    lines = [f"# {name}", "", f"source: `{os.path.basename(path)}` (ncu --metrics gpu__time_duration.sum "
             "--clock-control none; cold-cache, serialised launches: compare shares, not absolutes)", "",
             "| kernel | launches | mean us | total us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k[:90]}` | {len(v)} | {sum(v) / len(v):.2f} | {sum(v):.1f} | {sum(v) / total:.3f} |")
    os.makedirs(PROF, exist_ok=True)
    with open(os.path.join(PROF, f"{name}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("src")
    ap.add_argument("name")
    ap.add_argument("--launches", action="store_true")
    ap.add_argument("--config")
    ap.add_argument("--algo-bytes", type=float)
    a = ap.parse_args()
    if a.launches:
        summarise_launches(a.src, a.name)
    else:
        summarise_report(a.src, a.name, a.config, a.algo_bytes)


if __name__ == "__main__":
    main()
