"""ncu helper: one multi_head_dilated call at config-2 shapes (B=64, h=6, (512,2), bf16)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa  # noqa: E402

B, N, h, d = 64, 4096, 6, 64
D = h * d
cfg = dfa.AttentionConfig(N, 512, 2, h, d, dfa.AttentionConfig.spread_offsets(h, 2))
x = torch.randn((B, N, D), device="cuda", dtype=torch.bfloat16)
wq, wk, wv = (torch.randn((h, D, d), device="cuda", dtype=torch.bfloat16) / D ** 0.5 for _ in range(3))
wo = torch.randn((D, D), device="cuda", dtype=torch.bfloat16) / D ** 0.5
out = torch.empty_like(x)
for _ in range(3):
    dfa.multi_head_dilated(x, wq, wk, wv, wo, cfg, out=out)
torch.cuda.synchronize()
