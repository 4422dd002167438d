"""PCIe roofline for the e2e path: pinned H2D / D2H copy bandwidth alone and
concurrent, vs the zero-copy forward kernel (inputs read over PCIe in place)
and the full dfa_forward_host call."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa  # noqa: E402

MB = 1 << 20
n = 256 * MB
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
dv = torch.empty(n, dtype=torch.uint8, device="cuda")
dv2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


t = timed(lambda: dv.copy_(h, non_blocking=True))
print(f"H2D {n / t / 1e6:.1f} GB/s")
t = timed(lambda: h.copy_(dv, non_blocking=True))
print(f"D2H {n / t / 1e6:.1f} GB/s")


def both():
    ev = torch.cuda.Event()
    ev.record()
    with torch.cuda.stream(s1):
        s1.wait_event(ev)
        dv.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        s2.wait_event(ev)
        h2.copy_(dv2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


t = timed(both)
print(f"H2D+D2H concurrent: {2 * n / t / 1e6:.1f} GB/s total ({n / t / 1e6:.1f} each way)")

B, N, hh, d = 64, 4096, 6, 64
cfg = dfa.AttentionConfig(N, 512, 2, hh, d, dfa.AttentionConfig.spread_offsets(hh, 2))
hq, hk, hv = (torch.randn((B, N, hh, d)).to(torch.bfloat16).pin_memory() for _ in range(3))
o = torch.empty((B, N, hh, d), dtype=torch.bfloat16, device="cuda")
c = cfg._c()
t = timed(lambda: dfa._check(dfa.lib.dfa_forward(ctypes.byref(c), 1, B, hq.data_ptr(), hk.data_ptr(), hv.data_ptr(),
                                                 o.data_ptr(), None, torch.cuda.current_stream().cuda_stream)))
kept = 3 * B * N * hh * d * 2 // 2
print(f"zero-copy kernel (inputs over PCIe): {t:.2f} ms, {kept / t / 1e6:.1f} GB/s of kept rows")
ho = torch.empty_like(hq).pin_memory()
ws = dfa.Workspace(dfa.Workspace.bytes_for(cfg, "bf16", B))
t = timed(lambda: dfa.dfa_forward_host(hq, hk, hv, ho, cfg, ws))
print(f"dfa_forward_host e2e: {t:.2f} ms -> {B / t * 1e3:.0f} images/s; in {kept / 1e6:.0f} MB + out {ho.numel() * 2 / 1e6:.0f} MB")
t = timed(lambda: ho.copy_(o, non_blocking=True))
print(f"output D2H alone: {t:.2f} ms")
