"""Projection GEMMs of the multi-head layer (class split, config 2) under forced
tile widths vs auto: QKV [2 x 131072 x 384] @ [384 x 576], Wo [2 x 131072 x 192]
@ [192 x 384] with row-strided output."""
import sys, torch
sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa
M = 64 * 4096
A = torch.randn((2, M // 2, 384), device="cuda", dtype=torch.bfloat16)
W = torch.randn((2, 384, 576), device="cuda", dtype=torch.bfloat16) / 20
A2 = torch.randn((2, M // 2, 192), device="cuda", dtype=torch.bfloat16)
W2 = torch.randn((2, 192, 384), device="cuda", dtype=torch.bfloat16) / 14
out2 = torch.empty((M // 2, 2, 384), device="cuda", dtype=torch.bfloat16)  # rows 2t + g: row-strided class output
def t(fn, iters=20):
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
    for bn in (0, 192, 3192):
        dfa.lib.dfa_set_gemm_tile(bn)
        q = t(lambda: dfa.gemm(A, W))
        o = t(lambda: dfa.gemm(A2, W2, out=out2.transpose(0, 1)))
        line.append(f"bn={bn}: qkv {q:6.1f} wo {o:5.1f}")
    print(" | ".join(line), flush=True)
dfa.lib.dfa_set_gemm_tile(0)
