"""One config-4 forward cell (B = 64, h = 6, N = 4096) for ncu: python fwd_cell_once.py W R."""
import sys, torch
sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa
w, r = int(sys.argv[1]), int(sys.argv[2])
cfg = dfa.AttentionConfig(4096, w, r, 6, 64, dfa.AttentionConfig.spread_offsets(6, r))
q, k, v = (torch.randn((64, 4096, 6, 64), device="cuda", dtype=torch.bfloat16) for _ in range(3))
o = torch.empty_like(q)
for _ in range(3):
    dfa.dfa_forward(q, k, v, cfg, out=o)
torch.cuda.synchronize()
