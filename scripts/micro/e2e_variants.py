import os, subprocess, sys
CHILD = r'''
import sys, torch
sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa
B, N, h, d = 64, 4096, 6, 64
cfg = dfa.AttentionConfig(N, 512, 2, h, d, dfa.AttentionConfig.spread_offsets(h, 2))
hq, hk, hv = (torch.randn((B, N, h, d)).to(torch.bfloat16).pin_memory() for _ in range(3))
ho = torch.empty_like(hq).pin_memory()
ws = dfa.Workspace(dfa.Workspace.bytes_for(cfg, "bf16", B))
for _ in range(2): dfa.dfa_forward_host(hq, hk, hv, ho, cfg, ws)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(6): dfa.dfa_forward_host(hq, hk, hv, ho, cfg, ws)
e1.record(); torch.cuda.synchronize()
print(f"{64 * 6 / (e0.elapsed_time(e1) / 1e3):.0f} images/s")
'''
for lib in sys.argv[1:]:
    env = dict(os.environ, DFA_LIB_VARIANT=os.path.abspath(lib))
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print(os.path.basename(lib), r.stdout.strip() or r.stderr[-300:])
