"""Host-side cost per call (no sync inside the loop): dfa_forward and the
fused multi-branch call, B=64 h=6."""
import sys, time, torch
sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa
q, k, v = (torch.randn((64, 4096, 6, 64), device="cuda", dtype=torch.bfloat16) for _ in range(3))
o = torch.empty_like(q)
cfg2 = dfa.AttentionConfig(4096, 512, 2, 6, 64, [j % 2 for j in range(6)])
cfg = dfa.AttentionConfig(4096, 512, 1, 6, 64, [0] * 6)
br = [(512, 1), (1024, 2), (2048, 4), (4096, 8)]
for name, fn in (("dfa_forward", lambda: dfa.dfa_forward(q, k, v, cfg2, out=o)),
                 ("multibranch", lambda: dfa.dfa_forward_multibranch(q, k, v, cfg, br, out=o))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name}: host {1e6 * (t1 - t0) / 50:.1f} us per call")

# split: ctypes call alone (args prebuilt) vs the Python wrapper
import ctypes
c = cfg2._c()
c.value_dim = 64
sp = torch.cuda.current_stream().cuda_stream
args = (ctypes.byref(c), dfa._dtype_code(q), 64, q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), None, sp)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    dfa.lib.dfa_forward(*args)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"dfa_forward C-ABI only: {1e6 * (t1 - t0) / 50:.1f} us per call")
t0 = time.perf_counter()
for _ in range(50):
    cfg2._c()
t1 = time.perf_counter()
print(f"cfg._c(): {1e6 * (t1 - t0) / 50:.1f} us")
t0 = time.perf_counter()
for _ in range(50):
    torch.cuda.current_stream().cuda_stream
t1 = time.perf_counter()
print(f"current_stream: {1e6 * (t1 - t0) / 50:.1f} us")
t0 = time.perf_counter()
for _ in range(50):
    dfa._check_qkv(q, k, v, cfg2, "x")
t1 = time.perf_counter()
print(f"_check_qkv: {1e6 * (t1 - t0) / 50:.1f} us")
