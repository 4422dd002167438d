#!/usr/bin/env python3
"""Time profiling variants of libdfa.so (scripts/build_variant.sh) on the
BASELINE config-4 shapes; one subprocess per variant (ctypes loads once).

    python scripts/variants.py scripts/variants/libdfa_A.so ... [--cases 512:2,2048:1]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, sys, torch
sys.path.insert(0, sys.argv[1])
import paper_2403_09195_b200 as dfa
cases = [tuple(map(int, c.split(":"))) for c in sys.argv[2].split(",")]
N, h, d, B = 4096, 6, 64, 64
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn((B, N, h, d), device="cuda", dtype=torch.bfloat16, generator=g) for _ in range(3))
o = torch.empty_like(q)
ref = None
out = {}
for w, r in cases:
    cfg = dfa.AttentionConfig(N, w, r, h, d, dfa.AttentionConfig.spread_offsets(h, r))
    for _ in range(5):
        dfa.dfa_forward(q, k, v, cfg, out=o)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for rep in range(5):
        e0.record()
        for _ in range(20):
            dfa.dfa_forward(q, k, v, cfg, out=o)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 20)
    fl = 2 * dfa.flop_count(cfg).dilated_mults * B
    out[f"{w}:{r}"] = {"ms": best, "tflops": fl / best / 1e9}
print(json.dumps(out))
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--cases", default="512:2,1024:2,2048:1,4096:8")
    a = ap.parse_args()
    for lib in a.libs:
        env = dict(os.environ, DFA_LIB_VARIANT=os.path.abspath(lib))
        res = subprocess.run([sys.executable, "-c", CHILD, ROOT, a.cases], env=env, capture_output=True, text=True)
        line = res.stdout.strip().splitlines()[-1] if res.stdout.strip() else res.stderr[-400:]
        try:
            d = json.loads(line)
            print(os.path.basename(lib), " ".join(f"{k} {v['ms'] * 1e3:.1f}us {v['tflops']:.0f}TF" for k, v in d.items()))
        except ValueError:
            print(os.path.basename(lib), "FAILED", line)


if __name__ == "__main__":
    main()
