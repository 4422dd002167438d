"""A/B the backward across variant libraries at config 2 (one process per lib, interleaved)."""
import json, os, subprocess, sys
CHILD = r'''
import json, sys, torch
sys.path.insert(0, sys.argv[1])
import paper_2403_09195_b200 as dfa
B, N, h, d = 64, 4096, 6, 64
out = {}
import os
for w, r in [tuple(map(int, c.split(':'))) for c in os.environ.get('SHAPES', '512:2,256:2,256:1,512:4,1024:8').split(',')]:
    cfg = dfa.AttentionConfig(N, w, r, h, d, dfa.AttentionConfig.spread_offsets(h, r))
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v, do = (torch.randn((B, N, h, d), device="cuda", dtype=torch.bfloat16, generator=g) for _ in range(4))
    L = torch.empty((B, h, N), device="cuda")
    o = dfa.dfa_forward(q, k, v, cfg, lse=L)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    ws = torch.empty(B * h * N * 4 + 256, dtype=torch.uint8, device="cuda")
    f = lambda: dfa.dfa_backward(q, k, v, o, L, do, cfg, dq, dk, dv, workspace=ws)
    for _ in range(3): f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): f()
        e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) / 10)
    out[f"{w}:{r}"] = sorted(ts)[2]
    out[f"{w}:{r}:sum"] = float(dq.float().abs().sum() + dk.float().abs().sum() + dv.float().abs().sum())
    del q, k, v, do, L, o, dq, dk, dv
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
            print(lib, "FAILED", r.stderr[-800:]); continue
        for k, v in d.items():
            res.setdefault(os.path.basename(lib), {}).setdefault(k, []).append(v)
for lib, d in res.items():
    print(f"{lib:22s}", "  ".join(f"{k} {sorted(v)[len(v)//2]*1e3:6.1f}us" for k, v in d.items() if not k.endswith("sum")))
    print(" " * 22, "checksums", {k: round(v[0], 1) for k, v in d.items() if k.endswith("sum")})
