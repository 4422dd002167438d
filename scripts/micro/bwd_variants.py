"""Time dfa_backward of several libdfa builds (DFA_LIB_VARIANT) on config-4 shapes."""
import os, subprocess, sys
CHILD = r'''
import sys, torch
sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa
out = []
for w, r in ((512, 2), (256, 2), (1024, 4), (256, 1)):
    cfg = dfa.AttentionConfig(4096, w, r, 6, 64, [j % r for j in range(6)])
    q, k, v, do = (torch.randn((64, 4096, 6, 64), device="cuda", dtype=torch.bfloat16) for _ in range(4))
    L = torch.empty((64, 6, 4096), device="cuda")
    o = dfa.dfa_forward(q, k, v, cfg, lse=L)
    g = [torch.empty_like(q) for _ in range(3)]
    ws = torch.empty(64 * 6 * 4096 * 4 + 256, dtype=torch.uint8, device="cuda")
    for _ in range(3): dfa.dfa_backward(q, k, v, o, L, do, cfg, *g, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): dfa.dfa_backward(q, k, v, o, L, do, cfg, *g, workspace=ws)
    e1.record(); torch.cuda.synchronize()
    out.append(f"{w}:{r} {e0.elapsed_time(e1)/10*1e3:.0f}us")
print(" ".join(out))
'''
for lib in sys.argv[1:]:
    env = dict(os.environ, DFA_LIB_VARIANT=os.path.abspath(lib))
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print(os.path.basename(lib), r.stdout.strip() or r.stderr[-300:])
