#!/usr/bin/env python3
"""Softmax-region instruction mix and stall breakdown from an ncu report
(SASS source page): instructions executed per opcode class and per step,
stall samples by reason.  python scripts/ncu_softmax_mix.py REP [steps]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 0
KN = sys.argv[3] if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep] + (["-k", "regex:" + KN] if KN else []) + ["--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
ci = h.index("Instructions Executed")
si = h.index("Warp Stall Sampling (All Samples)")
reasons = [(i, x[6:]) for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
region, regions = "prologue", collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) < 5:
        continue
    src = r[1].strip()
    if "USETMAXREG" in src:
        region = src[:50]
    g = regions.setdefault(region, {"ops": collections.Counter(), "stall": collections.Counter(), "samples": 0})
    try:
        n = float(r[ci] or 0)
        s = float(r[si] or 0)
    except ValueError:
        continue
    op = src.split()[0] if not src.startswith("@") else src.split()[1]
    op = op.split(".")[0]
    g["ops"][op] += n
    g["samples"] += s
    for i, name in reasons:
        try:
            g["stall"][name] += float(r[i] or 0)
        except (ValueError, IndexError):
            pass
for reg, g in regions.items():
    tot = sum(g["ops"].values())
    if tot == 0:
        continue
    print(f"=== {reg}: {tot:.0f} warp-instr, {g['samples']:.0f} samples")
    st = sum(g["stall"].values()) or 1
    print("  stalls:", ", ".join(f"{k} {v / st:.0%}" for k, v in g["stall"].most_common(8)))
    for op, n in g["ops"].most_common(22):
        per = f"  {n / steps:8.1f}/step" if steps else ""
        print(f"  {op:12s} {n:12.0f} {n / tot:6.1%}{per}")
