"""Forward at the same work with h = 6 (128-B head column blocks of 768-B
token rows) vs h = 1 (contiguous 128-B rows): isolates the cost of the
strided per-head reads/writes."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa

def t(B, h, w, r):
    N, d = 4096, 64
    cfg = dfa.AttentionConfig(N, w, r, h, d, [j % r for j in range(h)])
    q, k, v = (torch.randn((B, N, h, d), device="cuda", dtype=torch.bfloat16) for _ in range(3))
    o = torch.empty_like(q)
    for _ in range(5):
        dfa.dfa_forward(q, k, v, cfg, out=o)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        dfa.dfa_forward(q, k, v, cfg, out=o)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    by = B * h * (2 * d * (N // r) * 3 + 2 * d * N)
    print(f"B={B} h={h} (w,r)=({w},{r}) {ms*1e3:.1f} us {by/ms/1e6:.0f} GB/s")

for w, r in ((512, 2), (256, 8), (2048, 1)):
    t(64, 6, w, r)
    t(384, 1, w, r)
