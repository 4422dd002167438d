#!/usr/bin/env python3
"""Per-kernel SASS instruction mix of the shipped libdfa.so (cuobjdump), the
evidence that the hot kernels run tcgen05 / TMA / TMEM code:
UTCHMMA / UTCQMMA (tcgen05.mma), UTCBAR (tcgen05.commit), UTMALDG / UTMASTG
(TMA load / store), LDTM / STTM (TMEM ld / st), MUFU.EX2, FFMA2 / FADD2.

    python scripts/sass_summary.py [--out profiles/r01_sass.md]
"""
import argparse
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UTMAPF", "LDTM", "STTM", "MUFU.EX2", "FFMA2", "FADD2",
        "FFMA", "HMMA", "SYNCS", "LDS", "STS", "LDG", "STG", "SHFL"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_2403_09195_b200", "libdfa.so"))
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_sass.md"))
    a = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", a.lib], capture_output=True, text=True, check=True).stdout
    arch = sorted(set(re.findall(r"arch = (sm_\w+)", sass)))
    funcs = re.split(r"\n\s*Function : ", sass)[1:]
    rows = []
    for f in funcs:
        name = f.split("\n", 1)[0].strip()
        demangled = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", f)
        cnt = collections.Counter()
        for op in ops:
            for k in KEYS:
                if op == k or op.startswith(k + "."):
                    cnt[k] += 1
        rows.append((demangled[:110], len(ops), cnt))
    with open(a.out, "w") as fh:
        fh.write(f"# SASS instruction mix of libdfa.so\n\n`cuobjdump -sass` of `{os.path.relpath(a.lib, ROOT)}`; "
                 f"target {', '.join(arch)}.  Static counts per kernel (instructions in the binary, not executed).\n\n")
        fh.write("| kernel | SASS lines | " + " | ".join(KEYS) + " |\n|---|---|" + "---|" * len(KEYS) + "\n")
        for name, n, cnt in sorted(rows, key=lambda r: -r[1]):
            fh.write(f"| `{name}` | {n} | " + " | ".join(str(cnt.get(k, 0)) for k in KEYS) + " |\n")
    print(open(a.out).read())


if __name__ == "__main__":
    sys.exit(main())
