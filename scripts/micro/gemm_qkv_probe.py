"""QKV-projection GEMM (batch 2 x [131072 x 384] @ [384 x 576]) at auto tiles: time only
(run under DFA_LIB_VARIANT for the probe builds)."""
import os, sys, torch
sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa
M, K, N = 64 * 4096, 384, 576
A = torch.randn((2, M // 2, K), device="cuda", dtype=torch.bfloat16)
w = torch.randn((2, K, N), device="cuda", dtype=torch.bfloat16) / K ** 0.5
Wo = torch.randn((2, 192, 384), device="cuda", dtype=torch.bfloat16)
A2 = torch.randn((2, M // 2, 192), device="cuda", dtype=torch.bfloat16)
W1 = torch.randn((384, 1536), device="cuda", dtype=torch.bfloat16)
X = torch.randn((M, 384), device="cuda", dtype=torch.bfloat16)
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
out = []
for name, fn, fl in (("qkv", lambda: dfa.gemm(A, w), 2 * M * K * N), ("wo", lambda: dfa.gemm(A2, Wo), 2 * M * 192 * 384),
                     ("w1", lambda: dfa.gemm(X, W1), 2 * M * 384 * 1536)):
    us = t(fn)
    out.append(f"{name} {us:6.1f}us {fl / us / 1e6:5.0f}TF")
print(os.path.basename(os.environ.get("DFA_LIB_VARIANT", "product")), " | ".join(out))
