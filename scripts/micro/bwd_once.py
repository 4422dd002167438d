"""One config-2 backward (plus warm-up) for ncu captures; library from DFA_LIB_VARIANT if set."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa
w, r = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "512:2").split(":"))
B, N, h = 64, 4096, 6
cfg = dfa.AttentionConfig(N, w, r, h, 64, dfa.AttentionConfig.spread_offsets(h, r))
q, k, v, do = (torch.randn((B, N, h, 64), device="cuda", dtype=torch.bfloat16) for _ in range(4))
L = torch.empty((B, h, N), device="cuda")
o = dfa.dfa_forward(q, k, v, cfg, lse=L)
g = [torch.empty_like(q) for _ in range(3)]
ws = torch.empty(B * h * N * 4 + 256, dtype=torch.uint8, device="cuda")
for _ in range(3):
    dfa.dfa_backward(q, k, v, o, L, do, cfg, *g, workspace=ws)
torch.cuda.synchronize()
