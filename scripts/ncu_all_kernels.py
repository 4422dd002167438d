#!/usr/bin/env python3
"""One launch of every kernel family in libdfa.so, for an ncu capture:

    ncu --set full --clock-control none -o gpurun_out/prof_all python scripts/ncu_all_kernels.py
    python scripts/ncu_all_kernels.py --summarize gpurun_out/prof_all.ncu-rep profiles/r01_kernels_ncu.md
"""
import csv
import io
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run():
    import torch

    import paper_2403_09195_b200 as dfa
    from paper_2403_09195_b200 import _lib, path_override

    g = torch.Generator(device="cuda").manual_seed(0)
    bf, f32 = torch.bfloat16, torch.float32
    N, h, d = 4096, 6, 64
    cfg = dfa.AttentionConfig(N, 512, 2, h, d, dfa.AttentionConfig.spread_offsets(h, 2))
    q, k, v, do = (torch.randn((64, N, h, d), device="cuda", dtype=bf, generator=g) for _ in range(4))
    L = torch.empty((64, h, N), device="cuda", dtype=f32)
    torch.cuda.synchronize()
    o = dfa.dfa_forward(q, k, v, cfg, lse=L)                                   # sm100 forward (+ lse)
    dfa.dfa_forward_multibranch(q[:16], k[:16], v[:16], cfg, [(512, 1), (2048, 4)])  # sm100 normal + merge
    dfa.dfa_backward(q, k, v, o, L, do, cfg)                                   # delta + tcgen05 backward
    c1 = dfa.AttentionConfig(N, 512, 2, 1, d, [0])
    x1 = [torch.randn((1, N, 1, d), device="cuda", dtype=f32, generator=g) for _ in range(3)]
    dfa.dfa_forward(*x1, c1)                                                   # SIMT fp32 (config 1)
    c3 = dfa.AttentionConfig(1200, 300, 3, h, d, dfa.AttentionConfig.spread_offsets(h, 3))
    x3 = [torch.randn((16, 1200, h, d), device="cuda", dtype=bf, generator=g) for _ in range(3)]
    dfa.dfa_forward(*x3, c3)                                                   # SIMT bf16 (general geometry)
    xf = [t.float() for t in (q[:4], k[:4], v[:4])]
    dfa.dfa_forward_multibranch(*xf, cfg, [(512, 2), (1024, 4)])               # SIMT branches + combine kernel
    Lf = torch.empty((4, h, N), device="cuda", dtype=f32)
    of = dfa.dfa_forward(*xf, cfg, lse=Lf)
    with path_override(_lib.DFA_PATH_SIMT):
        dfa.dfa_backward(*xf, of, Lf, do[:4].float(), cfg)                     # SIMT backward
    D = h * d
    x = torch.randn((64, N, D), device="cuda", dtype=bf, generator=g)
    s = D ** -0.5
    p = {"ln1_g": torch.ones(D), "ln1_b": torch.zeros(D), "wq": s * torch.randn(h, D, d), "wk": s * torch.randn(h, D, d),
         "wv": s * torch.randn(h, D, d), "wo": s * torch.randn(D, D), "bo": torch.zeros(D), "ln2_g": torch.ones(D),
         "ln2_b": torch.zeros(D), "w1": s * torch.randn(D, 4 * D), "b1": torch.zeros(4 * D),
         "w2": torch.randn(4 * D, D) / (4 * D) ** 0.5, "b2": torch.zeros(D)}
    p = {kk: vv.to("cuda", bf).contiguous() for kk, vv in p.items()}
    dfa.encoder_block_forward(x, p, cfg)                                       # LN, pack, GEMMs, strided core, GELU
    torch.cuda.synchronize()


METRICS = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "read MB"), ("dram__bytes_write.sum", "write MB"),
           ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
           ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor %"),
           ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU %"),
           ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue %"),
           ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
           ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid")]


def summarize(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ki = hdr.index("Kernel Name")
    idx = {m: hdr.index(m) for m, _ in METRICS if m in hdr}
    scale = {"dram__bytes_read.sum": 1, "dram__bytes_write.sum": 1}
    with open(out, "w") as fh:
        fh.write(f"# ncu `--set full` of every kernel family (one launch each)\n\nsource: `{os.path.basename(rep)}` "
                 "(`scripts/ncu_all_kernels.py`, `--clock-control none`; cuBLASLt GEMMs are library kernels).\n\n")
        fh.write("| kernel | " + " | ".join(lbl for _, lbl in METRICS) + " |\n|---|" + "---|" * len(METRICS) + "\n")
        for r in data:
            name = r[ki][:90]
            vals = []
            for m, _ in METRICS:
                if m not in idx:
                    vals.append("")
                    continue
                x = r[idx[m]]
                u = units[idx[m]]
                try:
                    f = float(x.replace(",", ""))
                    if m.startswith("dram__bytes"):
                        f = f * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(u, 1)
                    if m == "gpu__time_duration.sum":
                        f = f * {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(u, 1)
                    vals.append(f"{f:.1f}" if f < 1e5 else f"{f:.3g}")
                except ValueError:
                    vals.append(x)
            fh.write(f"| `{name}` | " + " | ".join(vals) + " |\n")
    print(open(out).read())


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--summarize":
        summarize(sys.argv[2], sys.argv[3])
    else:
        run()
