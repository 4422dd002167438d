"""ncu helper: one multibranch call (LongNet set) and its four single-branch calls, B=64 h=6."""
import sys, torch
sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa
q, k, v = (torch.randn((64, 4096, 6, 64), device="cuda", dtype=torch.bfloat16) for _ in range(3))
cfg = dfa.AttentionConfig(4096, 512, 1, 6, 64, [0] * 6)
ws = torch.empty(1 << 31, dtype=torch.uint8, device="cuda")
br = [(512, 1), (1024, 2), (2048, 4), (4096, 8)]
for _ in range(3):
    dfa.dfa_forward_multibranch(q, k, v, cfg, br, workspace=ws)
for w, r in br:
    c = dfa.AttentionConfig(4096, w, r, 6, 64, dfa.AttentionConfig.spread_offsets(6, r))
    dfa.dfa_forward(q, k, v, c)
torch.cuda.synchronize()
