#!/usr/bin/env python3
"""Record and decode the CTA-0 timeline of the tcgen05 kernel (dfa_forward_traced).

On the GPU box:  python scripts/trace_timeline.py run  [--w 512 --r 2 --batch 64]
Here:            python scripts/trace_timeline.py show gpurun_out/trace.npy
"""
import argparse
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CAP = 4096
NAMES = {1: "Q_ISSUE", 2: "KV_WAIT", 3: "KV_ISSUE", 4: "P_WAIT", 5: "P_READY", 6: "PV_ISSUED", 7: "QK_WAIT",
         8: "QK_ISSUED", 9: "S_WAIT", 10: "S_READY", 11: "MAX_DONE", 12: "EXP_DONE", 13: "P_ARRIVE", 14: "O_WAIT",
         15: "O_READY", 16: "STORE_ISSUED", 17: "QK_GOT", 18: "PV_GOT", 19: "Q_GOT"}
ROLES = ["producer", "mma", "softmax_A", "softmax_B", "epilogue", "pv"]


def run_mb(args):
    """Fused multi-branch kernel (dfa_set_multibranch_trace) on --set."""
    import torch

    import paper_2403_09195_b200 as dfa

    sets = {"longnet": [(512, 1), (1024, 2), (2048, 4), (4096, 8)], "long2": [(2048, 2), (4096, 4)],
            "r2set": [(256, 2), (512, 2), (1024, 4)]}
    br = sets[args.set]
    h = 6
    cfg = dfa.AttentionConfig(4096, 512, 1, h, 64, [0] * h)
    q, k, v = (torch.randn((args.batch, 4096, h, 64), device="cuda", dtype=torch.bfloat16) for _ in range(3))
    o = torch.empty_like(q)
    tr = torch.zeros(6 * CAP + 2048, dtype=torch.int64, device="cuda")
    for _ in range(3):
        dfa.dfa_forward_multibranch(q, k, v, cfg, br, out=o)
    dfa.lib.dfa_set_multibranch_trace(tr.data_ptr())
    dfa.dfa_forward_multibranch(q, k, v, cfg, br, out=o)
    dfa.lib.dfa_set_multibranch_trace(None)
    torch.cuda.synchronize()
    out = os.path.join(ROOT, "gpurun_out", f"trace_mb_{args.set}.npy")
    save_and_show(tr, out)


def save_and_show(tr, out):
    raw = tr.cpu().numpy().astype(np.uint64)
    np.save(out, raw[:6 * CAP])
    ct = raw[6 * CAP:].astype(np.int64).reshape(-1, 2)
    ct = ct[ct[:, 0] > 0]
    if len(ct):
        t0 = ct[:, 0].min()
        ends = (ct[:, 1] - t0) / 1e3
        print(f"per-CTA end (us): min {ends.min():.1f} median {np.median(ends):.1f} max {ends.max():.1f}; "
              f"start spread {(ct[:, 0].max() - t0) / 1e3:.1f} us")
    show(out)


def run(args):
    import torch

    import paper_2403_09195_b200 as dfa
    from paper_2403_09195_b200 import _lib

    h = 6
    offs = [j % args.r for j in range(h)]
    cfg = dfa.AttentionConfig(4096, args.w, args.r, h, 64, offs)
    q, k, v = (torch.randn((args.batch, 4096, h, 64), device="cuda", dtype=torch.bfloat16) for _ in range(3))
    o = torch.empty_like(q)
    tr = torch.zeros(6 * CAP + 2048, dtype=torch.int64, device="cuda")
    c = cfg._c()
    for _ in range(3):  # warm (clocks, L2 state)
        dfa.dfa_forward(q, k, v, cfg, out=o)
    dfa._check(dfa.lib.dfa_forward_traced(ctypes.byref(c), args.batch, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                          o.data_ptr(), tr.data_ptr(), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    out = os.path.join(ROOT, "gpurun_out", f"trace_w{args.w}_r{args.r}.npy")
    save_and_show(tr, out)


def decode(path):
    raw = np.load(path).astype(np.uint64)
    ev = {}
    for s, role in enumerate(ROLES):
        seg = raw[s * CAP:(s + 1) * CAP]
        seg = seg[seg != 0]
        ev[role] = [(int(x >> np.uint64(56)), int(x & np.uint64(0xFFFFFFFFFFFFFF))) for x in seg]
    t0 = min(e[0][1] for e in ev.values() if e)
    return {r: [(NAMES[c], t - t0) for c, t in e] for r, e in ev.items()}, t0


def spans(events, a, b):
    """durations from each event a to the next event b."""
    out, start = [], None
    for name, t in events:
        if name == a:
            start = t
        elif name == b and start is not None:
            out.append(t - start)
            start = None
    return np.array(out) if out else np.array([0])


def show(path):
    ev, _ = decode(path)
    end = max(t for e in ev.values() for _, t in e)
    print(f"CTA 0 timeline: {end} cycles total")
    for role in ("softmax_A", "softmax_B"):
        e = ev[role]
        n = sum(1 for x, _ in e if x == "S_READY")
        sw = spans(e, "S_WAIT", "S_READY")
        mx = spans(e, "S_READY", "MAX_DONE")
        ex = spans(e, "MAX_DONE", "EXP_DONE")
        pa = spans(e, "EXP_DONE", "P_ARRIVE")
        gap = spans(e, "P_ARRIVE", "S_WAIT")
        busy = mx.sum() + ex.sum() + pa.sum()
        print(f"{role}: {n} steps; per step mean: wait-S {sw.mean():.0f}, ld+max {mx.mean():.0f}, "
              f"exp {ex.mean():.0f}, tail {pa.mean():.0f}, between {gap.mean():.0f}; busy {busy / end:.1%} "
              f"(wait-S total {sw.sum() / end:.1%})")
    m, pv = ev["mma"], ev["pv"]
    print(f"qk issuer: q_full wait {spans(m, 'QK_WAIT', 'Q_GOT').mean():.0f} per unit, "
          f"k_full wait {spans(m, 'Q_GOT', 'QK_GOT').mean():.0f}, issue gaps {np.diff([t for n, t in m if n == 'QK_ISSUED']).mean():.0f}")
    pw = spans(pv, "P_WAIT", "P_READY")
    print(f"pv issuer: p-wait mean {pw.mean():.0f} (total {pw.sum() / end:.1%}), operands {spans(pv, 'P_READY', 'PV_GOT').mean():.0f}, "
          f"issue {spans(pv, 'PV_GOT', 'PV_ISSUED').mean():.0f}")
    pr = ev["producer"]
    kw = spans(pr, "KV_WAIT", "KV_ISSUE")
    print(f"producer: kv-empty wait mean {kw.mean():.0f} (total {kw.sum() / end:.1%})")
    ep = ev["epilogue"]
    ow = spans(ep, "O_WAIT", "O_READY")
    st = spans(ep, "O_READY", "STORE_ISSUED")
    print(f"epilogue: o-full wait mean {ow.mean():.0f} (total {ow.sum() / end:.1%}), "
          f"readout+store mean {st.mean():.0f}")
    # first few steps in detail
    for role in ("mma", "pv", "softmax_A", "softmax_B"):
        print(role, " ".join(f"{n}@{t}" for n, t in ev[role][:24]))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("cmd", choices=["run", "run_mb", "show"])
    ap.add_argument("--set", default="longnet")
    ap.add_argument("path", nargs="?")
    ap.add_argument("--w", type=int, default=512)
    ap.add_argument("--r", type=int, default=2)
    ap.add_argument("--batch", type=int, default=64)
    a = ap.parse_args()
    {"run": run, "run_mb": run_mb}[a.cmd](a) if a.cmd != "show" else show(a.path)
