"""Backward device time on one-block views (m <= 128: fused kernel, nb = 1)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa  # noqa: E402

B, N, h, d = 64, 4096, 6, 64
out = []
for w, r in ((256, 2), (512, 4), (1024, 8), (256, 4), (256, 8), (512, 8)):
    cfg = dfa.AttentionConfig(N, w, r, h, d, dfa.AttentionConfig.spread_offsets(h, r))
    q, k, v, do = (torch.randn((B, N, h, d), device="cuda", dtype=torch.bfloat16) for _ in range(4))
    L = torch.empty((B, h, N), device="cuda", dtype=torch.float32)
    o = dfa.dfa_forward(q, k, v, cfg, lse=L)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    ws = torch.empty(B * h * N * 4 + 256, dtype=torch.uint8, device="cuda")
    f = lambda: dfa.dfa_backward(q, k, v, o, L, do, cfg, dq, dk, dv, workspace=ws)  # noqa: E731
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        e0.record()
        for _ in range(10):
            f()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 10)
    out.append(f"({w},{r}) {best * 1e3:.1f}us")
print(" ".join(out))
