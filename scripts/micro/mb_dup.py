"""Fused kernel mechanics check: a duplicated single branch [(w,r),(w,r)]
(schedule = the single kernel's units, twice the steps) vs 2x dfa_forward."""
import sys, torch
sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa
B, N, h = 64, 4096, 6
q, k, v = (torch.randn((B, N, h, 64), device="cuda", dtype=torch.bfloat16) for _ in range(3))
o = torch.empty_like(q)
def t(fn, iters=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters): fn()
        e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) / iters)
    return sorted(ts)[2] * 1e3
for w, r in ((2048, 1), (1024, 1), (512, 1), (2048, 2)):
    cfg = dfa.AttentionConfig(N, w, r, h, 64, dfa.AttentionConfig.spread_offsets(h, r))
    br = [(w, r), (w, r)]
    tm = t(lambda: dfa.dfa_forward_multibranch(q, k, v, cfg, br, out=o))
    n = dfa.last_launch_count()
    ts = t(lambda: dfa.dfa_forward(q, k, v, cfg, out=o))
    print(f"({w},{r}) dup fused {tm:.1f} us ({n} launch) = {tm/2:.1f} per branch | single {ts:.1f} us")
