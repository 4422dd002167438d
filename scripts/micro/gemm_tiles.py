"""dfa_gemm at the config-2 layer shapes for every forced tile width (64 /
128 / 192 / 256; dfa_set_gemm_tile), CUDA events, warm: picks the dispatcher's
per-shape choice.   python scripts/micro/gemm_tiles.py"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa  # noqa: E402


def time_ms(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


bf = torch.bfloat16
M = 64 * 4096
for name, batch, m, n, k, bias, res, gelu in (("qkv cls", 2, M // 2, 576, 384, 0, 0, 0),
                                             ("wo cls +res", 2, M // 2, 384, 192, 1, 1, 0),
                                             ("qkv dense", 1, M, 1152, 384, 0, 0, 0),
                                             ("wo dense", 1, M, 384, 384, 0, 0, 0),
                                             ("w1 gelu", 1, M, 1536, 384, 1, 0, 1),
                                             ("w2 +res", 1, M, 384, 1536, 1, 1, 0)):
    A = torch.randn((batch, m, k), device="cuda", dtype=bf)
    B = torch.randn((batch, k, n), device="cuda", dtype=bf) / k ** 0.5
    bi = torch.randn((n,), device="cuda", dtype=bf) if bias else None
    C = torch.randn((batch, m, n), device="cuda", dtype=bf) if res else None
    out = torch.empty((batch, m, n), device="cuda", dtype=bf)
    line = f"{name:12s}"
    for bn in (0, 64, 128, 192, 256):
        dfa.lib.dfa_set_gemm_tile(bn)
        print(name, bn, flush=True) if len(sys.argv) > 1 else None
        ms = time_ms(lambda: dfa.gemm(A, B, bias=bi, c=C, gelu=bool(gelu), out=out))
        line += f"  bn{bn}: {ms:.4f}"
    dfa.lib.dfa_set_gemm_tile(0)
    print(line, flush=True)
