#!/usr/bin/env python3
"""BASELINE.json configs 1, 3, 4 (+ the LSE-combined branch set) on one B200.

    python scripts/sweeps.py [--out gpurun_out/sweeps.json] [--ncu]

config1  fp32 single head, N=4096, (512, 2), d=64, B=1 (SIMT validation path): latency
config3  6 encoder attention layers (fresh q/k/v each) x h=6 at (512, 2), batch 1..256,
         CUDA-graph captured: images/s = B / time(6 layers)
config4  (w, r) grid w in {256..4096}, r in {1, 2, 4, 8}, B=64, h=6, offsets j mod r:
         ms, TFLOP/s (2 x dilated_mults), algorithmic GB/s, roofline fraction of the
         attainable min(peak, AI x HBM) -- and the LSE-combined LongNet-style set
--ncu    one cold launch per config4 case (for an ncu --metrics pass over the script)
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2403_09195_b200 as dfa  # noqa: E402


def peaks():
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return p["hbm_gbs"], p["bf16_tflops"]
    except (OSError, KeyError, ValueError):
        return 6650.0, 1590.0


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


def cfg_for(N, w, r, h, d=64):
    return dfa.AttentionConfig(N, w, r, h, d, dfa.AttentionConfig.spread_offsets(h, r))


def config1():
    """fp32 single head, B = 1: a latency workload, so the 50 calls are
    replayed from a CUDA graph (the Python/ctypes launch path would otherwise
    be what is timed)."""
    N, d = 4096, 64
    q, k, v = (torch.randn((1, N, 1, d), device="cuda") for _ in range(3))
    cfg = cfg_for(N, 512, 2, 1)
    o = torch.empty_like(q)
    dfa.dfa_forward(q, k, v, cfg, out=o)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(50):
                dfa.dfa_forward(q, k, v, cfg, out=o, stream=s)
    torch.cuda.current_stream().wait_stream(s)
    ms = time_ms(g.replay, iters=10) / 50
    eager = time_ms(lambda: dfa.dfa_forward(q, k, v, cfg, out=o), iters=50)
    fc = dfa.flop_count(cfg)
    return {"config": "config1 fp32 B=1 h=1 N=4096 (512,2) d=64", "path": "simt f32 (split form)", "us": ms * 1e3,
            "us_eager_python_launch": eager * 1e3, "gflops": 2 * fc.dilated_mults / (ms / 1e3) / 1e9}


def config3():
    N, h, d, L = 4096, 6, 64, 6
    cfg = cfg_for(N, 512, 2, h)
    rows = []
    for B in (1, 2, 4, 8, 16, 32, 64, 128, 256):
        layers = [[torch.randn((B, N, h, d), device="cuda", dtype=torch.bfloat16) for _ in range(3)] for _ in range(L)]
        outs = [torch.empty_like(layers[0][0]) for _ in range(L)]

        def run():
            for (q, k, v), o in zip(layers, outs):
                dfa.dfa_forward(q, k, v, cfg, out=o)

        run()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for (q, k, v), o in zip(layers, outs):
                    dfa.dfa_forward(q, k, v, cfg, out=o, stream=s)
        torch.cuda.current_stream().wait_stream(s)
        ms = time_ms(g.replay, iters=max(5, 200 // B))
        fl = 2 * dfa.flop_count(cfg).dilated_mults * B * L
        rows.append({"B": B, "ms_6_layers": ms, "images_per_s": B / (ms / 1e3), "tflops": fl / (ms / 1e3) / 1e12})
        del layers, outs, g
        torch.cuda.empty_cache()
    return {"config": "config3 6 layers x h=6 (512,2) bf16, CUDA graph of 6 launches", "rows": rows}


def config4(ncu=False):
    N, h, d, B = 4096, 6, 64, 64
    hbm, tc = peaks()
    q, k, v = (torch.randn((B, N, h, d), device="cuda", dtype=torch.bfloat16) for _ in range(3))
    o = torch.empty_like(q)
    rows = []
    for w in (256, 512, 1024, 2048, 4096):
        for r in (1, 2, 4, 8):
            cfg = cfg_for(N, w, r, h)
            if ncu:
                dfa.dfa_forward(q, k, v, cfg, out=o)
                continue
            ms = time_ms(lambda: dfa.dfa_forward(q, k, v, cfg, out=o))
            fl = 2 * dfa.flop_count(cfg).dilated_mults * B
            by = B * h * (2 * d * (N // r) * 3 + 2 * d * N)
            ai = fl / by
            attain = min(tc, ai * hbm / 1e3)
            tf = fl / (ms / 1e3) / 1e12
            rows.append({"w": w, "r": r, "ms": ms, "tflops": tf, "GBps": by / (ms / 1e3) / 1e9, "AI": ai,
                         "attainable_tflops": attain, "frac_of_attainable": tf / attain, "frac_of_tensor_peak": tf / tc,
                         "bound": "tensor" if ai * hbm / 1e3 >= tc else "hbm"})
    if ncu:
        return None
    # LSE-combined LongNet-style set (extension): 4 branch kernels + combine
    branches = [(512, 1), (1024, 2), (2048, 4), (4096, 8)]
    cfg = cfg_for(N, 512, 1, h)
    ws = torch.empty(1 << 31, dtype=torch.uint8, device="cuda")
    ms = time_ms(lambda: dfa.dfa_forward_multibranch(q, k, v, cfg, branches, out=o, workspace=ws))
    fl = sum(2 * dfa.flop_count(cfg_for(N, w, r, h)).dilated_mults for w, r in branches) * B
    combo = {"branches": branches, "ms": ms, "tflops": fl / (ms / 1e3) / 1e12, "launches": dfa.last_launch_count()}
    return {"config": "config4 (w,r) sweep B=64 h=6 bf16", "rows": rows, "lse_combined_set": combo}


def config4_backward():
    """dfa_backward over the config-4 (w, r) grid (B = 64, h = 6, bf16): the
    tcgen05 kernels for m = w/r multiple of 128, SIMT otherwise.  FLOP = 2.5 x
    the forward's (S, dP, dV, dK, dQ; the long-m pair recomputes S / dP, so its
    executed FLOPs are 3.5 x)."""
    N, h, d, B = 4096, 6, 64, 64
    q, k, v, do = (torch.randn((B, N, h, d), device="cuda", dtype=torch.bfloat16) for _ in range(4))
    L = torch.empty((B, h, N), device="cuda", dtype=torch.float32)
    ws = torch.empty(B * h * N * 4 + 256, dtype=torch.uint8, device="cuda")
    g = [torch.empty_like(q) for _ in range(3)]
    rows = []
    for w in (256, 512, 1024, 2048, 4096):
        for r in (1, 2, 4, 8):
            cfg = cfg_for(N, w, r, h)
            o = dfa.dfa_forward(q, k, v, cfg, lse=L)
            m = w // r
            iters = 3 if m % 128 else 10
            ms = time_ms(lambda: dfa.dfa_backward(q, k, v, o, L, do, cfg, *g, workspace=ws), iters=iters, warmup=1)
            fl = 2.5 * 2 * dfa.flop_count(cfg).dilated_mults * B
            rows.append({"w": w, "r": r, "m": m, "ms": ms, "tflops": fl / (ms / 1e3) / 1e12,
                         "path": "tcgen05 fused" if m in (128, 256) else ("tcgen05 dkdv+dq" if m % 128 == 0 else (
                             "tcgen05 fused (packed segments)" if 128 % m == 0 and m >= 16 else "simt"))})
    return {"config": "config4 backward (w,r) sweep B=64 h=6 bf16", "rows": rows}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweeps.json"))
    ap.add_argument("--ncu", action="store_true")
    ap.add_argument("--only", choices=["config1", "config3", "config4", "config4bwd"], default=None)
    a = ap.parse_args()
    if a.ncu:
        config4(ncu=True)
        return
    fns = {"config1": config1, "config4": config4, "config3": config3, "config4bwd": config4_backward}
    res = {"gpu": torch.cuda.get_device_name(0)}
    for name, fn in fns.items():
        if a.only in (None, name):
            res[name] = fn()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)
    if "config1" in res:
        print(json.dumps(res["config1"]))
    for r in res.get("config4", {}).get("rows", []):
        print(f"w={r['w']:5d} r={r['r']} {r['ms']:.3f} ms {r['tflops']:7.1f} TF {r['GBps']:7.0f} GB/s "
              f"{r['frac_of_attainable']:.2f} of attainable ({r['bound']})")
    if "config4" in res:
        print("combined", res["config4"]["lse_combined_set"])
    for r in res.get("config4bwd", {}).get("rows", []):
        print(f"bwd w={r['w']:5d} r={r['r']} m={r['m']:4d} {r['ms']:.3f} ms {r['tflops']:7.1f} TF  {r['path']}")
    for r in res.get("config3", {}).get("rows", []):
        print(f"B={r['B']:4d} {r['ms_6_layers']:.3f} ms/6 layers {r['images_per_s']:9.0f} images/s {r['tflops']:.0f} TF")


if __name__ == "__main__":
    main()
