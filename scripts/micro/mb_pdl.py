"""Fused multi-branch launch timing: back-to-back events with and without PDL
(DFA_PDL is read once per process, so run twice)."""
import sys, torch
sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa
SETS = {"longnet": [(512, 1), (1024, 2), (2048, 4), (4096, 8)], "long2": [(2048, 2), (4096, 4)]}
q, k, v = (torch.randn((64, 4096, 6, 64), device="cuda", dtype=torch.bfloat16) for _ in range(3))
o = torch.empty_like(q)
cfg = dfa.AttentionConfig(4096, 512, 1, 6, 64, [0] * 6)
for name, br in SETS.items():
    for _ in range(3):
        dfa.dfa_forward_multibranch(q, k, v, cfg, br, out=o)
    torch.cuda.synchronize()
    res = []
    for n in (1, 10):
        ts = []
        for rep in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(n):
                dfa.dfa_forward_multibranch(q, k, v, cfg, br, out=o)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / n)
        res.append(sorted(ts)[3] * 1e3)
    print(name, "single launch %.1f us, back-to-back x10 %.1f us/launch" % tuple(res))
