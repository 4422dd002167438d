#!/usr/bin/env python3
"""Host-side checks of the fused multi-branch kernel (csrc/dfa_mb_sm100.cu).

1. The schedule: `dfa_multibranch_plan` returns the work-unit descriptors the
   kernel runs (built by the same C++ code, no GPU needed).  `check_plan`
   verifies that they cover every output row of every head exactly once, that
   each (row, branch) pair the extension oracle would use sees every key of its
   segment among the slot's steps for that branch, that rows no branch selects
   are flagged for exact zeros, and that the step bookkeeping the roles share
   (tile order, per-slot step lists, first / last tiles) is consistent.
2. The mbarrier protocol: every role loop of dfa_mb_sm100_kernel as a Python
   generator (async TMA / MMA completions immediate), the dynamic-claim ring
   included, run under random interleavings over a random sequence of claimed
   units -- no deadlock, every parity wait at most one phase away.

    python scripts/protocol_model_mb.py --N 4096 --h 6 --branches 512:1,1024:2,2048:4,4096:8
"""
import argparse
import ctypes
import os
import random
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from protocol_model import Bar, ParityHazard  # noqa: E402

KBM = KBN = 128
KSB, KKV, KQ, KSCHED, KCONS = 3, 3, 2, 6, 15
EARLY_FREE = False  # model a buggy consumer that frees its ring slot as soon as it took the unit


class RingOverwrite(AssertionError):
    pass


DESC = np.dtype({
    "names": ["j", "n_tiles", "steps", "qt", "first", "last", "cls", "sel", "anysel", "gamma", "tile", "sn", "sstep"],
    "formats": ["<i4", "<i4", "<i4", ("<i4", 2), ("<i4", 2), ("<i4", 2), ("<i2", (2, 8)), ("u1", (2, 8)),
                ("u1", 2), ("<i4", 8), ("<u4", 64), ("<i4", 2), ("<u4", (2, 64))],
    "offsets": [0, 4, 8, 12, 20, 28, 36, 68, 84, 88, 120, 376, 384],
    "itemsize": 896,
})


def plan(N, h, B, branches, grid=148):
    """branches: [(w, r, offsets[h])].  Returns (descs, R, gr) or raises."""
    import paper_2403_09195_b200 as dfa
    from paper_2403_09195_b200 import _lib

    w0, r0, o0 = branches[0]
    cfg = dfa.AttentionConfig(N, w0, r0, h, 64, list(o0))
    c = cfg._c()
    keep, bs = [], []
    for w, r, offs in branches:
        arr = (ctypes.c_int64 * h)(*offs)
        keep.append(arr)
        bs.append(_lib.DfaBranch(w, r, ctypes.cast(arr, ctypes.POINTER(ctypes.c_int64))))
    barr = (_lib.DfaBranch * len(bs))(*bs)
    nd, R, grl, db = (ctypes.c_int32() for _ in range(4))
    st = dfa.lib.dfa_multibranch_plan(ctypes.byref(c), len(bs), barr, B, grid, None, 0, ctypes.byref(nd),
                                      ctypes.byref(R), ctypes.byref(grl), ctypes.byref(db))
    dfa._check(st)
    assert db.value == DESC.itemsize, (db.value, DESC.itemsize)
    buf = np.zeros(nd.value * db.value, dtype=np.uint8)
    dfa._check(dfa.lib.dfa_multibranch_plan(ctypes.byref(c), len(bs), barr, B, grid, buf.ctypes.data, buf.nbytes,
                                            ctypes.byref(nd), ctypes.byref(R), ctypes.byref(grl), ctypes.byref(db)))
    return buf.view(DESC), R.value, 1 << grl.value


def slot_rows(d, s, R, gr, N):
    """Output rows of slot s: list of (row_in_tile, n)."""
    out = []
    if d["qt"][s] < 0:
        return out
    TR = N // R
    G = KBM // gr
    for g in range(G):
        for rin in range(gr):
            t = d["qt"][s] + rin
            if t < TR:
                out.append((g * gr + rin, int(t * R + d["cls"][s][g])))
    return out


def check_plan(descs, R, gr, N, h, branches):
    """Raises AssertionError on any schedule defect."""
    G = KBM // gr
    covered = np.zeros((h, N), dtype=np.int32)
    for d in descs:
        j = int(d["j"])
        tiles = [int(x) for x in d["tile"][: d["n_tiles"]]]
        # shared step order: per tile, slot A then slot B
        order = []
        for ti, wd in enumerate(tiles):
            mask = (wd >> 28) & 3
            for s in range(2):
                if (mask >> s) & 1:
                    order.append((ti, s))
        assert len(order) == d["steps"]
        for s in range(2):
            mine = [i for i, (ti, ss) in enumerate(order) if ss == s]
            assert d["sn"][s] == len(mine)
            for q, idx in enumerate(mine):
                e = int(d["sstep"][s][q])
                ti = order[idx][0]
                assert e >> 23 == idx, "per-slot step index"
                assert (e & 0xFFFFF) == (tiles[ti] & 0xFFFFFF) and ((e >> 20) & 7) == ((tiles[ti] >> 24) & 7)
            tis = [order[i][0] for i in mine]
            assert d["first"][s] == (tis[0] if tis else -1) and d["last"][s] == (tis[-1] if tis else -1)
        for s in range(2):
            rows = slot_rows(d, s, R, gr, N)
            if d["qt"][s] < 0:
                continue
            # key ranges this slot sees per branch
            seen = {}
            for q in range(d["sn"][s]):
                e = int(d["sstep"][s][q])
                seen.setdefault((e >> 20) & 7, []).append(e & 0xFFFFF)
            for rt, n in rows:
                covered[j, n] += 1
                g = rt // gr
                any_sel = False
                for k, (w, r, offs) in enumerate(branches):
                    sel = n % r == offs[j]
                    assert sel == bool((d["sel"][s][k] >> g) & 1), "selection bits"
                    if not sel:
                        continue
                    any_sel = True
                    m, T = w // r, N // r
                    tk = n // r
                    lo = (tk // m) * m
                    hi = min(lo + m, T)
                    starts = seen.get(k, [])
                    have = np.zeros(hi - lo, dtype=bool)
                    for tp in starts:
                        a, b = max(tp, lo), min(tp + KBN, hi)
                        if a < b:
                            have[a - lo:b - lo] = True
                    assert have.all(), f"row {n} head {j} branch {k}: keys missing"
                assert any_sel == bool((d["anysel"][s] >> g) & 1), "anysel bits"
    assert (covered == 1).all(), f"rows covered {covered.min()}..{covered.max()} times"


# ------------------------------------------------------------- protocol model
def run_protocol(descs, seq, seed=0):
    """seq: descriptor indices the CTA claims, in order.  None = OK, else the blocked waits."""
    B = dict(q_full=[Bar(f"q_full{i}", 1) for i in range(KQ)], q_empty=[Bar(f"q_empty{i}", 1) for i in range(KQ)],
             k_full=[Bar(f"k_full{i}", 1) for i in range(KKV)], k_empty=[Bar(f"k_empty{i}", 1) for i in range(KKV)],
             v_full=[Bar(f"v_full{i}", 1) for i in range(KKV)], v_empty=[Bar(f"v_empty{i}", 1) for i in range(KKV)],
             s_full=[[Bar(f"s_full{s}{b}", 1) for b in range(KSB)] for s in range(2)],
             p_full=[Bar(f"p_full{b}", KBM) for b in range(KSB)],
             s_free=[Bar(f"s_free{b}", 1) for b in range(KSB)], pv_done=[Bar(f"pv_done{s}", 1) for s in range(2)],
             o_full=[Bar(f"o_full{s}", 1) for s in range(2)], o_empty=[Bar(f"o_empty{s}", KBM) for s in range(2)],
             stat_full=[Bar(f"stat_full{s}", KBM) for s in range(2)],
             stat_empty=[Bar(f"stat_empty{s}", KBM) for s in range(2)],
             sched_full=[Bar(f"sched_full{i}", 1) for i in range(KSCHED)],
             sched_empty=[Bar(f"sched_empty{i}", KCONS) for i in range(KSCHED)])
    ring = [None] * KSCHED
    held = {}  # consumer role -> ring slot whose descriptor it is still reading
    claims = list(seq) + [None]  # None = the end sentinel
    D = lambda slot: descs[ring[slot]]  # noqa: E731

    def take(n, arrivals, who):
        """Consumer: free the previous unit's slot, wait for unit n; returns its ring slot."""
        if n > 0 and not EARLY_FREE:
            held.pop(who, None)
            B["sched_empty"][(n - 1) % KSCHED].arrive(arrivals)
        slot = n % KSCHED
        yield ("wait", B["sched_full"][slot], n // KSCHED + 1)
        held[who] = slot  # read until the role takes its next unit
        if EARLY_FREE:
            B["sched_empty"][slot].arrive(arrivals)
        return slot

    def producer():
        i = g = 0
        for n, e in enumerate(claims):
            qs = i % KQ
            yield ("wait", B["q_empty"][qs], i // KQ)
            slot = n % KSCHED
            yield ("wait", B["sched_empty"][slot], n // KSCHED)
            if slot in held.values():
                raise RingOverwrite(f"descriptor slot {slot} overwritten while read by {held}")
            ring[slot] = e
            B["sched_full"][slot].arrive()  # the descriptor's bulk copy completes with it
            if e is None:
                return
            d = descs[e]
            if d["n_tiles"] == 0:
                continue
            B["q_full"][qs].arrive()
            i += 1
            for t in range(d["n_tiles"]):
                st = g % KKV
                yield ("wait", B["k_empty"][st], g // KKV)
                B["k_full"][st].arrive()
                g += 1

    def producer_v():
        g = 0
        for n in range(len(claims)):
            slot = yield from take(n, 1, "v")
            if ring[slot] is None:
                return
            for t in range(D(slot)["n_tiles"]):
                st = g % KKV
                yield ("wait", B["v_empty"][st], g // KKV)
                B["v_full"][st].arrive()
                g += 1

    def qk_issuer():
        b = steps = gs = i = 0
        for n in range(len(claims)):
            slot = yield from take(n, 1, "qk")
            if ring[slot] is None:
                return
            d = D(slot)
            if d["n_tiles"] == 0:
                continue
            qs = i & 1
            yield ("wait", B["q_full"][qs], (i >> 1) + 1)
            i += 1
            for t in range(d["n_tiles"]):
                mask = (int(d["tile"][t]) >> 28) & 3
                yield ("wait", B["k_full"][gs % KKV], gs // KKV + 1)
                for sl in range(2):
                    if not (mask >> sl) & 1:
                        continue
                    if steps >= KSB:
                        yield ("wait", B["s_free"][b], steps // KSB)
                    B["s_full"][sl][b].arrive()
                    b = (b + 1) % KSB
                    steps += 1
                B["k_empty"][gs % KKV].arrive()
                gs += 1
            B["q_empty"][qs].arrive()

    def pv_issuer():
        b = steps = gs = 0
        oc = [0, 0]
        for n in range(len(claims)):
            slot = yield from take(n, 1, "pv")
            if ring[slot] is None:
                return
            d = D(slot)
            for t in range(d["n_tiles"]):
                mask = (int(d["tile"][t]) >> 28) & 3
                have_v = False
                for sl in range(2):
                    if not (mask >> sl) & 1:
                        continue
                    yield ("wait", B["p_full"][b], steps // KSB + 1)
                    if t == d["first"][sl]:
                        yield ("wait", B["o_empty"][sl], oc[sl])
                    if not have_v:
                        yield ("wait", B["v_full"][gs % KKV], gs // KKV + 1)
                        have_v = True
                    B["pv_done"][sl].arrive()
                    B["s_free"][b].arrive()
                    if t == d["last"][sl]:
                        B["o_full"][sl].arrive()
                        oc[sl] += 1
                    b = (b + 1) % KSB
                    steps += 1
                B["v_empty"][gs % KKV].arrive()
                gs += 1

    def softmax(s):
        use = [0] * KSB
        pvc = steps = published = 0
        kbase = 0
        for n in range(len(claims)):
            slot = yield from take(n, 4, f"softmax{s}")  # four warps per slot, lane 0 of each arrives
            if ring[slot] is None:
                return
            d = D(slot)
            k_unit = kbase
            kbase += int(d["steps"])
            if d["first"][s] < 0:
                continue
            for q in range(d["sn"][s]):
                here = int(d["sstep"][s][q]) >> 23
                b = (k_unit + here) % KSB
                yield ("wait", B["s_full"][s][b], use[b] + 1)
                use[b] += 1
                if steps > 0:
                    yield ("wait", B["pv_done"][s], pvc + 1)
                    pvc += 1
                steps += 1
                B["p_full"][b].arrive(KBM)
            if published > 0:
                yield ("wait", B["stat_empty"][s], published)
            B["stat_full"][s].arrive(KBM)
            published += 1

    def epilogue():
        par = [0, 0]
        for n in range(len(claims)):
            slot = yield from take(n, 4, "epi")
            if ring[slot] is None:
                return
            d = D(slot)
            for s in range(2):
                if d["qt"][s] < 0 or d["first"][s] < 0:
                    continue
                yield ("wait", B["o_full"][s], par[s] + 1)
                yield ("wait", B["stat_full"][s], par[s] + 1)
                par[s] += 1
                B["stat_empty"][s].arrive(KBM)
                B["o_empty"][s].arrive(KBM)

    roles = {"producer": producer(), "producer_v": producer_v(), "qk": qk_issuer(), "pv": pv_issuer(),
             "softmax_A": softmax(0), "softmax_B": softmax(1), "epilogue": epilogue()}
    rnd = random.Random(seed)
    blocked = {name: next(gen, None) for name, gen in roles.items()}
    names = list(roles)
    while True:
        progress = False
        if seed:
            rnd.shuffle(names)
        for name in names:
            w = blocked[name]
            while w is not None and w[1].done(w[2]):
                w = next(roles[name], None)
                progress = True
            blocked[name] = w
        if all(w is None for w in blocked.values()):
            return None
        if not progress:
            return {nm: (w[1].name, w[2], w[1].phase) for nm, w in blocked.items() if w is not None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=4096)
    ap.add_argument("--h", type=int, default=6)
    ap.add_argument("--branches", default="512:1,1024:2,2048:4,4096:8")
    ap.add_argument("--seeds", type=int, default=4)
    a = ap.parse_args()
    brs = []
    for x in a.branches.split(","):
        w, r = map(int, x.split(":"))
        brs.append((w, r, [j % r for j in range(a.h)]))
    descs, R, gr = plan(a.N, a.h, 2, brs)
    check_plan(descs, R, gr, a.N, a.h, brs)
    print(f"plan ok: {len(descs)} units, R = {R}, {gr} rows per class group, "
          f"{int(descs['steps'].sum())} steps per image")
    rnd = random.Random(0)
    for seed in range(a.seeds):
        seq = [rnd.randrange(len(descs)) for _ in range(40)]
        res = run_protocol(descs, seq, seed)
        print(f"protocol seed {seed}: {'ok' if res is None else res}")


if __name__ == "__main__":
    main()
