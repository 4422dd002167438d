import sys, torch
sys.path.insert(0, '.')
import paper_2403_09195_b200 as dfa
B, N, h, d = 64, 4096, 6, 64
D = h * d
cfg = dfa.AttentionConfig(N, 512, 2, h, d, dfa.AttentionConfig.spread_offsets(h, 2))
x = torch.randn((B, N, D), device="cuda", dtype=torch.bfloat16)
s = D ** -0.5
p = {"ln1_g": torch.ones(D), "ln1_b": torch.zeros(D), "wq": s * torch.randn(h, D, d), "wk": s * torch.randn(h, D, d),
     "wv": s * torch.randn(h, D, d), "wo": s * torch.randn(D, D), "bo": torch.zeros(D), "ln2_g": torch.ones(D),
     "ln2_b": torch.zeros(D), "w1": s * torch.randn(D, 4 * D), "b1": torch.zeros(4 * D),
     "w2": torch.randn(4 * D, D) / (4 * D) ** 0.5, "b2": torch.zeros(D)}
p = {k: v.to("cuda", torch.bfloat16).contiguous() for k, v in p.items()}
for _ in range(3):
    y = dfa.encoder_block_forward(x, p, cfg)
torch.cuda.synchronize()
