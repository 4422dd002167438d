"""Zero-copy in + out timing of the forward (inputs and O over PCIe in place),
for the current library (DFA_LIB_VARIANT selects a variant build)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa  # noqa: E402

B, N, h, d = 64, 4096, 6, 64
cfg = dfa.AttentionConfig(N, 512, 2, h, d, dfa.AttentionConfig.spread_offsets(h, 2))
hq, hk, hv = (torch.randn((B, N, h, d)).to(torch.bfloat16).pin_memory() for _ in range(3))
ho = torch.empty_like(hq).pin_memory()
c = cfg._c()


def zc2():
    dfa._check(dfa.lib.dfa_forward(ctypes.byref(c), 1, B, hq.data_ptr(), hk.data_ptr(), hv.data_ptr(), ho.data_ptr(),
                                   None, torch.cuda.current_stream().cuda_stream))


zc2()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    zc2()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"zero-copy in + out: {ms:.2f} ms -> {B / ms * 1e3:.0f} images/s")
