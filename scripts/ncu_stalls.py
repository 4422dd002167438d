#!/usr/bin/env python3
"""Per-source-line stall breakdown from an ncu report (needs -lineinfo).
    python scripts/ncu_stalls.py REP.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
KN = sys.argv[3] if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep] + (["-k", "regex:" + KN] if KN else []) + ["--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
h = rows[hi]
reasons = [(i, x) for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
agg = []
tot_reason = {}
for r in rows[hi + 1:]:
    if len(r) > 40 and r[0] != "":
        try:
            v = float(r[4])
        except ValueError:
            continue
        rs = {}
        for i, name in reasons:
            try:
                x = float(r[i])
            except ValueError:
                x = 0
            if x:
                rs[name[6:]] = x
                tot_reason[name[6:]] = tot_reason.get(name[6:], 0) + x
        agg.append((v, r[0], r[1].strip()[:70], rs))
tot = sum(a[0] for a in agg)
print(f"total samples {tot:.0f}; by reason:",
      ", ".join(f"{k} {v / tot:.1%}" for k, v in sorted(tot_reason.items(), key=lambda kv: -kv[1])[:10]))
for v, l, s, rs in sorted(agg, reverse=True)[:n]:
    top = ", ".join(f"{k}:{int(x)}" for k, x in sorted(rs.items(), key=lambda kv: -kv[1])[:3])
    print(f"{v:6.0f} L{l:5s} {s:70s} | {top}")
