"""ncu helper: the w1 + b1 + GELU GEMM at config 2 (M = 262144, N = 1536, K = 384)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa  # noqa: E402

bf = torch.bfloat16
M = 64 * 4096
A = torch.randn((M, 384), device="cuda", dtype=bf)
B = torch.randn((384, 1536), device="cuda", dtype=bf) / 20
bi = torch.randn((1536,), device="cuda", dtype=bf)
out = torch.empty((M, 1536), device="cuda", dtype=bf)
for _ in range(2):
    dfa.gemm(A, B, bias=bi, gelu=True, out=out)
torch.cuda.synchronize()
