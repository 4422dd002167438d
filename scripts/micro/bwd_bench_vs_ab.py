"""Backward at config 2 timed two ways: bench.py's f_rows loop (20 back-to-back
calls on a side stream) and bwd_ab's (10 calls, median of 5, default stream)."""
import sys, time, torch
sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa
B, N, h, d = 64, 4096, 6, 64
cfg = dfa.AttentionConfig(N, 512, 2, h, d, dfa.AttentionConfig.spread_offsets(h, 2))
q, k, v, do = (torch.randn((B, N, h, d), device="cuda", dtype=torch.bfloat16) for _ in range(4))
L = torch.empty((B, h, N), device="cuda")
o = dfa.dfa_forward(q, k, v, cfg, lse=L)
g = [torch.empty_like(q) for _ in range(3)]
ws = torch.empty(B * h * N * 4 + 256, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for label, stream, n in (("side stream x20", s, 20), ("default x10", None, 10), ("side stream x20", s, 20)):
    for _ in range(3): dfa.dfa_backward(q, k, v, o, L, do, cfg, *g, workspace=ws, stream=stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    (e0.record(stream) if stream else e0.record())
    for _ in range(n): dfa.dfa_backward(q, k, v, o, L, do, cfg, *g, workspace=ws, stream=stream)
    (e1.record(stream) if stream else e1.record())
    host = (time.perf_counter() - t0) / n * 1e6
    torch.cuda.synchronize()
    print(f"{label}: {e0.elapsed_time(e1) / n * 1e3:.1f} us/call (host issue {host:.0f} us/call)")
