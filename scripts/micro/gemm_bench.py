"""Layer GEMM shapes at config 2 (B = 64 images, N = 4096, D = 384, h = 6,
(512, 2) offset-class split, hidden 1536): dfa_gemm (tcgen05) vs
torch.matmul (cuBLAS) on the same shapes, CUDA events, warm, back to back.
Prints ms, TFLOP/s and algorithmic GB/s per shape.

    python scripts/micro/gemm_bench.py [--out gpurun_out/gemm_bench.json]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2403_09195_b200 as dfa  # noqa: E402


def time_ms(fn, iters=20, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "gemm_bench.json"))
    a = ap.parse_args()
    bf = torch.bfloat16
    M = 64 * 4096
    shapes = [  # name, batch, M, N, K, bias, residual, gelu
        ("qkv class-split (r=2)", 2, M // 2, 576, 384, False, False, False),
        ("wo class-split (r=2) +bo +res", 2, M // 2, 384, 192, True, True, False),
        ("qkv dense", 1, M, 1152, 384, False, False, False),
        ("wo dense", 1, M, 384, 384, False, False, False),
        ("w1 +b1 +gelu", 1, M, 1536, 384, True, False, True),
        ("w2 +b2 +res", 1, M, 384, 1536, True, True, False),
    ]
    rows = []
    for name, batch, m, n, k, bias, res, gelu in shapes:
        A = torch.randn((batch, m, k), device="cuda", dtype=bf)
        B = torch.randn((batch, k, n), device="cuda", dtype=bf) / k ** 0.5
        bi = torch.randn((n,), device="cuda", dtype=bf) if bias else None
        C = torch.randn((batch, m, n), device="cuda", dtype=bf) if res else None
        out = torch.empty((batch, m, n), device="cuda", dtype=bf)
        ms = time_ms(lambda: dfa.gemm(A, B, bias=bi, c=C, gelu=gelu, out=out))

        def torch_fn():
            y = torch.matmul(A, B)
            if bias:
                y = y + bi
            if res:
                y = y + C
            if gelu:
                y = torch.nn.functional.gelu(y)
            return y

        def torch_mm():
            return torch.matmul(A, B, out=out)

        ms_t = time_ms(torch_fn)
        ms_mm = time_ms(torch_mm)
        fl = 2.0 * batch * m * n * k
        by = 2.0 * batch * (m * k + k * n + m * n + (m * n if res else 0))
        rows.append({"shape": name, "batch": batch, "M": m, "N": n, "K": k, "ms": ms, "tflops": fl / ms / 1e9,
                     "GBps": by / ms / 1e6, "torch_ms": ms_t, "torch_matmul_only_ms": ms_mm})
        print(f"{name:34s} dfa {ms:.4f} ms {fl / ms / 1e9:7.1f} TF {by / ms / 1e6:6.0f} GB/s | torch {ms_t:.4f} ms"
              f" (matmul alone {ms_mm:.4f})")
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump({"gpu": torch.cuda.get_device_name(0), "rows": rows}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
