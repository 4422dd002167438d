"""One forward shape, a few launches (for ncu captures): fwd_once.py W R [B]."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa  # noqa: E402

w, r = int(sys.argv[1]), int(sys.argv[2])
B = int(sys.argv[3]) if len(sys.argv) > 3 else 16
N, h = 4096, 6
q, k, v = (torch.randn((B, N, h, 64), device="cuda", dtype=torch.bfloat16) for _ in range(3))
cfg = dfa.AttentionConfig(N, w, r, h, 64, dfa.AttentionConfig.spread_offsets(h, r))
o = torch.empty_like(q)
for _ in range(4):
    dfa.dfa_forward(q, k, v, cfg, out=o)
torch.cuda.synchronize()
