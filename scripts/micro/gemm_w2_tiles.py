"""w2 of the encoder block (M = 262144, K = 1536, N = 384, bias + residual) and
w1 (K = 384, N = 1536, bias + GELU) under forced tile widths vs auto."""
import sys, torch
sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa
M = 64 * 4096
H = torch.randn((M, 1536), device="cuda", dtype=torch.bfloat16)
W2 = torch.randn((1536, 384), device="cuda", dtype=torch.bfloat16) / 40
b2 = torch.randn(384, device="cuda", dtype=torch.bfloat16)
R = torch.randn((M, 384), device="cuda", dtype=torch.bfloat16)
X = torch.randn((M, 384), device="cuda", dtype=torch.bfloat16)
W1 = torch.randn((384, 1536), device="cuda", dtype=torch.bfloat16) / 20
b1 = torch.randn(1536, device="cuda", dtype=torch.bfloat16)
def t(fn, iters=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters): fn()
        e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) / iters)
    return sorted(ts)[2] * 1e3
for rep in range(2):
    line = []
    for bn in (0, 128, 192, 256):
        dfa.lib.dfa_set_gemm_tile(bn)
        a = t(lambda: dfa.gemm(H, W2, bias=b2, c=R))
        b = t(lambda: dfa.gemm(X, W1, bias=b1, gelu=True))
        line.append(f"bn={bn}: w2 {a:6.1f} w1 {b:6.1f}")
    print(" | ".join(line), flush=True)
dfa.lib.dfa_set_gemm_tile(0)
