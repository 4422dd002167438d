"""The class-split QKV GEMM (batch 2 x [131072 x 384] @ [384 x 576], row-strided A)
under forced tile widths vs auto, plus cuBLAS on the same shape."""
import sys, torch
sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa
M, K, N = 64 * 4096, 384, 576
x = torch.randn((M, K), device="cuda", dtype=torch.bfloat16)
a = x.view(M // 2, 2 * K)  # row-strided class view: rows 2t + g
w = torch.randn((2, K, N), device="cuda", dtype=torch.bfloat16) / K ** 0.5
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
A = torch.stack([a[:, :K], a[:, K:]])  # contiguous copy for the torch reference only
fl = 2 * M * K * N
for rep in range(2):
    for bn in (0, 64, 128, 192, 256):
        dfa.lib.dfa_set_gemm_tile(bn)
        us = t(lambda: dfa.gemm(A, w))
        print(f"bn={bn:3d}: {us:6.1f} us {fl / us / 1e6:6.0f} TF")
    dfa.lib.dfa_set_gemm_tile(0)
    us = t(lambda: torch.matmul(A, w))
    print(f"cuBLAS : {us:6.1f} us {fl / us / 1e6:6.0f} TF")
