"""ncu helper: the fused kernel on a branch set whose schedule equals the
single-branch kernel's (long2 = {(2048,2),(4096,4)}) + the two single calls."""
import sys, torch
sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa
q, k, v = (torch.randn((64, 4096, 6, 64), device="cuda", dtype=torch.bfloat16) for _ in range(3))
cfg = dfa.AttentionConfig(4096, 2048, 2, 6, 64, [0] * 6)
br = [(2048, 2), (4096, 4)]
for _ in range(3):
    dfa.dfa_forward_multibranch(q, k, v, cfg, br)
for w, r in br:
    c = dfa.AttentionConfig(4096, w, r, 6, 64, dfa.AttentionConfig.spread_offsets(6, r))
    dfa.dfa_forward(q, k, v, c)
torch.cuda.synchronize()
