"""Time dfa_forward_multibranch on branch sets (B=64, h=6): fused single kernel
vs per-branch launches.  python scripts/micro/mb_time.py"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa  # noqa: E402
from paper_2403_09195_b200 import _lib, multibranch_mode  # noqa: E402

SETS = {"longnet": [(512, 1), (1024, 2), (2048, 4), (4096, 8)],
        "longnet3": [(512, 1), (1024, 2), (2048, 4)],
        "r2set": [(256, 2), (512, 2), (1024, 4)],
        "long2": [(2048, 2), (4096, 4)]}
B, N, h = 64, 4096, 6
q, k, v = (torch.randn((B, N, h, 64), device="cuda", dtype=torch.bfloat16) for _ in range(3))
o = torch.empty_like(q)
cfg = dfa.AttentionConfig(N, 512, 1, h, 64, [0] * h)
ws = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
res = {}


def timed(fn, iters=20):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / iters)
    return best


for name, br in SETS.items():
    fl = sum(4 * 64 * N * w // (r * r) for w, r in br) * h * B
    tf_l, tp_l = [], []
    for rep in range(8):  # interleaved A/B (clock / power drift): medians
        tf_l.append(timed(lambda: dfa.dfa_forward_multibranch(q, k, v, cfg, br, out=o, workspace=ws), 10))
        n_f = dfa.last_launch_count()
        with multibranch_mode(_lib.DFA_MB_PER_BRANCH):
            tp_l.append(timed(lambda: dfa.dfa_forward_multibranch(q, k, v, cfg, br, out=o, workspace=ws), 10))
    t_f, t_p = sorted(tf_l)[4], sorted(tp_l)[4]
    res[name] = {"fused_ms": t_f, "fused_tf": fl / t_f / 1e9, "fused_launches": n_f,
                 "per_branch_ms": t_p, "per_branch_tf": fl / t_p / 1e9}
    print(f"{name:9s} fused {t_f*1e3:7.1f} us {fl/t_f/1e9:6.0f} TF ({n_f} launch) | per-branch {t_p*1e3:7.1f} us "
          f"{fl/t_p/1e9:6.0f} TF")
print(json.dumps(res))
