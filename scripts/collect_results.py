"""Render a directory of bench.py JSON lines as a markdown results table.

    python scripts/collect_results.py gpurun_out/final > profiles/r01_results.md
"""
import glob
import json
import os
import sys


def load(path):
    for line in reversed(open(path).read().strip().splitlines()):
        line = line.strip()
        if line.startswith("{"):
            try:
                return json.loads(line)
            except json.JSONDecodeError:
                return None
    return None


def fmt(v, nd=3):
    if v is None:
        return "—"
    if isinstance(v, float):
        return f"{v:.{nd}g}"
    return str(v)


def main():
    d = sys.argv[1]
    rows = []
    for p in sorted(glob.glob(os.path.join(d, "*.json"))):
        r = load(p)
        if not r or "roofline" not in r:
            continue
        rf = r["roofline"] or {}
        cpu = r.get("cpu_baseline") or {}
        e2e = r.get("e2e") or {}
        clk = r.get("clocks") or {}
        rows.append((os.path.basename(p)[:-5], r["config"].get("workload", "")[:70], fmt(r["value"]), r["unit"],
                     fmt(r["ms_per_step"], 4), rf.get("bound"), fmt(rf.get("achieved")), rf.get("unit"),
                     fmt(rf.get("frac")), fmt(cpu.get("value")), fmt(e2e.get("value")),
                     f"{clk.get('sm_mhz')} {','.join(clk.get('reasons', []))}"))
    print("| run | workload | value | unit | ms/step | bound | achieved | roofline unit | frac | cpu oracle | e2e | SM MHz |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for row in rows:
        print("| " + " | ".join(str(x) for x in row) + " |")
    # round-2 sub-records: sustained (power-capped), multi-epoch launches, IT beside AR
    print()
    print("| run | sustained value | sustained SM MHz | multi-epoch value (epochs/launch, frac) | IT prefix+search | IT linear scan | AR / IT scan |")
    print("|---|---|---|---|---|---|---|")
    for p in sorted(glob.glob(os.path.join(d, "*.json"))):
        r = load(p)
        if not r or "roofline" not in r:
            continue
        sus = r.get("sustained") or {}
        me = r.get("multi_epoch") or {}
        it = r.get("it_comparison") or {}
        print(f"| {os.path.basename(p)[:-5]} | {fmt(sus.get('value'))} | {(sus.get('clocks') or {}).get('sm_mhz', '—')} | "
              f"{fmt(me.get('value'))}" + (f" ({me.get('epochs_per_launch')}, {fmt(me.get('frac'))})" if me else "") +
              f" | {fmt((it.get('it') or {}).get('value'))} | {fmt((it.get('it_scan') or {}).get('value'))} | "
              f"{fmt(it.get('ar_over_it_scan'))} |")


if __name__ == "__main__":
    main()
