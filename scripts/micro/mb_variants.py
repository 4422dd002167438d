"""A/B the fused multi-branch kernel across variant libraries (one process
per lib, interleaved rounds): python scripts/micro/mb_variants.py LIB..."""
import json, os, subprocess, sys
CHILD = r'''
import json, sys, torch
sys.path.insert(0, sys.argv[1])
import paper_2403_09195_b200 as dfa
SETS = {"longnet": [(512, 1), (1024, 2), (2048, 4), (4096, 8)], "long2": [(2048, 2), (4096, 4)],
        "r2set": [(256, 2), (512, 2), (1024, 4)]}
B, N, h = 64, 4096, 6
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn((B, N, h, 64), device="cuda", dtype=torch.bfloat16, generator=g) for _ in range(3))
o = torch.empty_like(q)
cfg = dfa.AttentionConfig(N, 512, 1, h, 64, [0] * h)
ws = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
out = {}
for name, br in SETS.items():
    for _ in range(3):
        dfa.dfa_forward_multibranch(q, k, v, cfg, br, out=o, workspace=ws)
    torch.cuda.synchronize()
    ts = []
    for rep in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            dfa.dfa_forward_multibranch(q, k, v, cfg, br, out=o, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 10)
    out[name] = sorted(ts)[2]
print(json.dumps(out))
'''
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
res = {}
for rnd in range(3):
    for lib in sys.argv[1:]:
        env = dict(os.environ, DFA_LIB_VARIANT=os.path.abspath(lib))
        r = subprocess.run([sys.executable, "-c", CHILD, ROOT], env=env, capture_output=True, text=True)
        try:
            d = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception:
            print(lib, "FAILED", r.stderr[-500:]); continue
        for k, v in d.items():
            res.setdefault(os.path.basename(lib), {}).setdefault(k, []).append(v)
for lib, d in res.items():
    print(f"{lib:22s}", "  ".join(f"{k} {sorted(v)[len(v)//2]*1e3:7.1f}us" for k, v in d.items()))
