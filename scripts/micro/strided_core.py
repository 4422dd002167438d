"""Core time on fused-projection layouts: the offset-class call of the
multi-head layer (qkv [64, 2048, 3, 3, 64], r = 1, w = 256) vs the dense
strided call (qkv [64, 4096, 3, 6, 64], (512, 2)) vs contiguous q/k/v."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2403_09195_b200 as dfa  # noqa: E402


def t(fn, it=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it * 1e3


B = 64
qkv_c = torch.randn((B, 2048, 3, 3, 64), device="cuda", dtype=torch.bfloat16)
cfg_c = dfa.AttentionConfig(2048, 256, 1, 3, 64, [0, 0, 0])
o_c = torch.empty((B, 2048, 3, 64), device="cuda", dtype=torch.bfloat16)
print(f"class call (strided, r=1): {t(lambda: dfa.dfa_forward_strided(qkv_c, cfg_c, out=o_c)):.1f} us")
q, k, v = (qkv_c[:, :, i].contiguous() for i in range(3))
print(f"class call (contiguous q/k/v): {t(lambda: dfa.dfa_forward(q, k, v, cfg_c, out=o_c)):.1f} us")
qkv_d = torch.randn((B, 4096, 3, 6, 64), device="cuda", dtype=torch.bfloat16)
cfg_d = dfa.AttentionConfig(4096, 512, 2, 6, 64, dfa.AttentionConfig.spread_offsets(6, 2))
o_d = torch.empty((B, 4096, 6, 64), device="cuda", dtype=torch.bfloat16)
print(f"dense strided (512,2): {t(lambda: dfa.dfa_forward_strided(qkv_d, cfg_d, out=o_d)):.1f} us")
