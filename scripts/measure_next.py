#!/usr/bin/env python3
"""Measurement of the SURVEY §8(f) rows on one B200 (CUDA events, warm,
inputs resident, >L2 working sets):

  backward   dfa_backward at config 2 (B=64, N=4096, h=6, d=64, (512, 2), bf16):
             algorithmic FLOP = 2.5 x forward (S recompute, dP, dV, dK, dQ = 5
             GEMM-shaped products vs 2), bytes = q,k,v,o,dO,lse read + dq,dk,dv written
  multihead  dfa_multi_head_dilated at config 2 shapes (x [64, 4096, 384] bf16);
             "tflops" counts executed FLOPs (offset-class split: projections / r),
             "tflops_dense_equivalent" the dense layer's
  block      dfa_encoder_block_forward (D=384, h=6, hidden=1536), B=64
  encoder6   six blocks back to back (the SAM-Lightening encoder depth), images/s

    python scripts/measure_next.py [--out gpurun_out/next.json]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
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
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "next.json"))
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--only", choices=["backward"], default=None)
    a = ap.parse_args()
    B, N, h, d, w, r = a.batch, 4096, 6, 64, 512, 2
    D, hidden = h * d, 4 * h * d
    cfg = dfa.AttentionConfig(N, w, r, h, d, dfa.AttentionConfig.spread_offsets(h, r))
    g = torch.Generator(device="cuda").manual_seed(0)
    bf = torch.bfloat16
    res = {"gpu": torch.cuda.get_device_name(0), "batch": B}
    fwd_flop = 2 * dfa.flop_count(cfg).dilated_mults * B

    # ---- backward
    q, k, v, do = (torch.randn((B, N, h, d), device="cuda", dtype=bf, generator=g) for _ in range(4))
    L = torch.empty((B, h, N), device="cuda", dtype=torch.float32)
    o = dfa.dfa_forward(q, k, v, cfg, lse=L)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    ws = torch.empty(B * h * N * 4 + 256, dtype=torch.uint8, device="cuda")
    ms = time_ms(lambda: dfa.dfa_backward(q, k, v, o, L, do, cfg, dq, dk, dv, workspace=ws), iters=5)
    kept = B * h * (N // r) * d * 2
    by = 5 * kept + B * h * (N // r) * 4 + 3 * B * N * h * d * 2
    res["backward"] = {"ms": ms, "tflops": 2.5 * fwd_flop / ms / 1e9, "GBps": by / ms / 1e6,
                       "forward_ms": time_ms(lambda: dfa.dfa_forward(q, k, v, cfg, out=o, lse=L)),
                       "path": "delta kernel + fused tcgen05 backward (m = w / r = %d)" % (w // r)}
    del q, k, v, do, o, dq, dk, dv, L
    if a.only == "backward":
        os.makedirs(os.path.dirname(a.out), exist_ok=True)
        json.dump(res, open(a.out, "w"), indent=1)
        print(json.dumps(res, indent=1))
        return

    # ---- multi-head layer
    x = torch.randn((B, N, D), device="cuda", dtype=bf, generator=g)
    wq, wk, wv = (torch.randn((h, D, d), device="cuda", dtype=bf, generator=g) / D ** 0.5 for _ in range(3))
    wo = torch.randn((D, D), device="cuda", dtype=bf, generator=g) / D ** 0.5
    out = torch.empty_like(x)
    need = 4 * B * N * D * 2 + (40 << 20)
    wsp = torch.empty(need, dtype=torch.uint8, device="cuda")
    ms = time_ms(lambda: dfa.multi_head_dilated(x, wq, wk, wv, wo, cfg, out=out, workspace=wsp))
    # executed FLOPs: the bf16 layer runs per offset class (r > 1), so the
    # projections do 1/r of the dense layer's multiply-adds
    dense_proj = 2 * B * N * D * D * 4
    proj_flop = dense_proj // r
    res["multihead"] = {"ms": ms, "images_per_s": B / ms * 1e3, "tflops": (proj_flop + fwd_flop) / ms / 1e9,
                        "tflops_dense_equivalent": (dense_proj + fwd_flop) / ms / 1e9,
                        "launches": dfa.last_launch_count()}

    # ---- encoder block / 6 blocks
    s = 1.0 / D ** 0.5
    p = {"ln1_g": torch.ones(D), "ln1_b": torch.zeros(D), "wq": s * torch.randn(h, D, d), "wk": s * torch.randn(h, D, d),
         "wv": s * torch.randn(h, D, d), "wo": s * torch.randn(D, D), "bo": torch.zeros(D), "ln2_g": torch.ones(D),
         "ln2_b": torch.zeros(D), "w1": s * torch.randn(D, hidden), "b1": torch.zeros(hidden),
         "w2": torch.randn(hidden, D) / hidden ** 0.5, "b2": torch.zeros(D)}
    p = {kk: vv.to("cuda", bf).contiguous() for kk, vv in p.items()}
    wsb = torch.empty(7 * B * N * D * 2 + 2 * B * N * hidden * 2 + (40 << 20), dtype=torch.uint8, device="cuda")
    y = torch.empty_like(x)
    ms = time_ms(lambda: dfa.encoder_block_forward(x, p, cfg, out=y, workspace=wsb), iters=10)
    blk_flop = proj_flop + fwd_flop + 2 * 2 * B * N * D * hidden
    res["block"] = {"ms": ms, "images_per_s": B / ms * 1e3, "tflops": blk_flop / ms / 1e9,
                    "tflops_dense_equivalent": (blk_flop - proj_flop + dense_proj) / ms / 1e9,
                    "launches": dfa.last_launch_count()}
    bufs = [x, y]

    def six():
        for i in range(6):
            dfa.encoder_block_forward(bufs[i % 2], p, cfg, out=bufs[(i + 1) % 2], workspace=wsb)

    ms = time_ms(six, iters=5)
    res["encoder6"] = {"ms": ms, "images_per_s": B / ms * 1e3, "tflops": 6 * blk_flop / ms / 1e9,
                       "tflops_dense_equivalent": 6 * (blk_flop - proj_flop + dense_proj) / ms / 1e9}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
