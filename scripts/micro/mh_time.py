"""multi_head_dilated at config 2 (B = 64, (512, 2), bf16): time per call."""
import sys, torch
sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa
B, N, h, d = 64, 4096, 6, 64
D = h * d
cfg = dfa.AttentionConfig(N, 512, 2, h, d, dfa.AttentionConfig.spread_offsets(h, 2))
x = torch.randn((B, N, D), device="cuda", dtype=torch.bfloat16)
wq, wk, wv = (torch.randn((h, D, d), device="cuda", dtype=torch.bfloat16) / D ** 0.5 for _ in range(3))
wo = torch.randn((D, D), device="cuda", dtype=torch.bfloat16) / D ** 0.5
out = torch.empty_like(x)
f = lambda: dfa.multi_head_dilated(x, wq, wk, wv, wo, cfg, out=out)
for _ in range(3): f()
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): f()
    e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) / 20)
print(f"multi-head {sorted(ts)[2] * 1e3:.1f} us")
