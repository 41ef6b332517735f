"""Per-opcode (and per address range) executed-instruction histogram of one kernel from an
ncu report's SASS source page:  python scripts/ncu_sass_hist.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
lines = out.splitlines()
hdr_i = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[hdr_i:]))))
ops, total = Counter(), 0
seq = []
for r in rows:
    try:
        n = int(r["Instructions Executed"])
    except (KeyError, ValueError):
        continue
    op = r["Source"].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    o = o.split(".")[0]
    ops[o] += n
    total += n
    seq.append((r["Address"], n, r["Source"].strip()))
print(f"total warp instructions executed: {total}")
for o, n in ops.most_common(top):
    print(f"{o:12s} {n:14d} {n / total:6.3f}")
if "--hot" in sys.argv:
    for a, n, s in sorted(seq, key=lambda x: -x[1])[:60]:
        print(a[-5:], n, s[:70])

if "--blocks" in sys.argv:
    # basic-block-like runs: consecutive instructions with the same execution count
    runs = []
    for a, n, src in seq:
        if runs and runs[-1][2] == n:
            runs[-1][1] = a
            runs[-1][3] += 1
            runs[-1][4].append(src)
        else:
            runs.append([a, a, n, 1, [src]])
    runs.sort(key=lambda r: -r[2] * r[3])
    for a0, a1, n, k, srcs in runs[:25]:
        ops = Counter(s.split()[1 if s.split()[0].startswith("@") else 0].split(".")[0] for s in srcs if s.split())
        print(f"{a0[-5:]}-{a1[-5:]} x{n:>9d} len {k:4d} total {n * k:>11d}  {dict(ops.most_common(6))}")
