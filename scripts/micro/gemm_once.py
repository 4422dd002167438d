"""ncu helper: one dfa_gemm launch per layer shape of gemm_bench.py (config 2)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa  # noqa: E402

bf = torch.bfloat16
M = 64 * 4096
for batch, m, n, k, bias, res, gelu in ((2, M // 2, 576, 384, 0, 0, 0), (1, M, 384, 384, 0, 0, 0),
                                        (1, M, 1536, 384, 1, 0, 1), (1, M, 384, 1536, 1, 1, 0)):
    A = torch.randn((batch, m, k), device="cuda", dtype=bf)
    B = torch.randn((batch, k, n), device="cuda", dtype=bf) / k ** 0.5
    bi = torch.randn((n,), device="cuda", dtype=bf) if bias else None
    C = torch.randn((batch, m, n), device="cuda", dtype=bf) if res else None
    out = torch.empty((batch, m, n), device="cuda", dtype=bf)
    for _ in range(2):
        dfa.gemm(A, B, bias=bi, c=C, gelu=bool(gelu), out=out)
    torch.cuda.synchronize()
