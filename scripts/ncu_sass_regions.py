#!/usr/bin/env python3
"""Stall samples per SASS instruction, grouped by warp-role region (regions
start at each USETMAXREG).  python scripts/ncu_sass_regions.py REP [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
reasons = [(i, x[6:]) for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
region = "prologue"
groups = {}
for r in rows[hi + 1:]:
    if len(r) < 5:
        continue
    src = r[1].strip()
    if "USETMAXREG" in src:
        region = src.split()[1] + " " + src.split()[-2].strip(",;") if "ALLOC" in src else src
        region = src[:60]
    try:
        v = float(r[2])
    except ValueError:
        continue
    rs = {}
    for i, name in reasons:
        try:
            x = float(r[i])
        except (ValueError, IndexError):
            x = 0
        if x:
            rs[name] = x
    groups.setdefault(region, []).append((v, r[0][-5:], src[:60], rs))
tot = sum(v for g in groups.values() for v, *_ in g)
for reg, items in groups.items():
    s = sum(v for v, *_ in items)
    print(f"\n=== region after [{reg}] : {s:.0f} samples ({s / tot:.1%})")
    for v, a, src, rs in sorted(items, reverse=True)[:n]:
        top = ", ".join(f"{k}:{int(x)}" for k, x in sorted(rs.items(), key=lambda kv: -kv[1])[:3])
        print(f"  {v:6.0f} {a} {src:60s} | {top}")
