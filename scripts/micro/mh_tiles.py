"""multi_head_dilated (config-2 shapes) under forced GEMM tile widths (dfa_set_gemm_tile)."""
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
ref = dfa.multi_head_dilated(x, wq, wk, wv, wo, cfg)
def t(iters=20):
    for _ in range(3):
        dfa.multi_head_dilated(x, wq, wk, wv, wo, cfg, out=out)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            dfa.multi_head_dilated(x, wq, wk, wv, wo, cfg, out=out)
        e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / iters)
    return best
for rep in range(2):
    for bn in (0, 64, 128, 192, 256):
        dfa.lib.dfa_set_gemm_tile(bn)
        ms = t()
        err = (out.float() - ref.float()).abs().max().item()
        print(f"bn={bn}: {ms*1e3:.1f} us  (max|diff| vs auto {err:.2e})")
    dfa.lib.dfa_set_gemm_tile(0)
