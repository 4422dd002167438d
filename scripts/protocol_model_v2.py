#!/usr/bin/env python3
"""Executable model of dfa_sm100_v2_kernel's mbarrier protocol (one CTA).

Same method as protocol_model.py (roles as generators, parity-checked waits,
round-robin / shuffled scheduling, deadlock = no role can progress), for the
four-slot kernel: per-slot S buffers, round-robin step order over slot
groups, per-slot Q stages.  Also checks the data side of the step order:
every step of slot s reads the ring stage holding key tile kt0_s + rho, and
each slot's tiles cover its rows' segments.

    python scripts/protocol_model_v2.py --N 4096 --w 512 --r 2 --h 6 --B 64
"""
import argparse
import random

from protocol_model import Bar, ParityHazard

KBM, KBN, SLOTS = 128, 64, 4
UNIT = SLOTS * KBM
KKV = 6


def make_unit(p, u):
    j, bp = u % p["h"], u // p["h"]
    blk, b = bp % p["n_blocks"], bp // p["n_blocks"]
    t0 = blk * UNIT
    m, T = p["m"], p["T"]
    kv_lo = (t0 // m) * m
    kt0, ln, segs = [], [], []
    for s in range(SLOTS):
        r0, r1 = t0 + s * KBM, min(t0 + s * KBM + KBM, T)
        if r0 < r1:
            lo, hi = (r0 // m) * m, min(((r1 - 1) // m + 1) * m, T)
            kt0.append((lo - kv_lo) // KBN)
            ln.append(-(-(hi - kv_lo) // KBN) - kt0[-1])
            segs.append((lo, hi))
        else:
            kt0.append(0)
            ln.append(0)
            segs.append(None)
    return dict(b=b, j=j, t0=t0, kv_lo=kv_lo, kt0=kt0, len=ln, rounds=max(ln), segs=segs)


def active(x, s, rho):
    return 0 <= s < SLOTS and rho < x["len"][s]


def lead(x, s, rho):
    return active(x, s, rho) and (s == 0 or x["kt0"][s] != x["kt0"][s - 1] or not active(x, s - 1, rho))


def last(x, s, rho):
    return active(x, s, rho) and (s == SLOTS - 1 or x["kt0"][s + 1] != x["kt0"][s] or not active(x, s + 1, rho))


def units(p, cta):
    return list(range(cta, p["n_units"], p["grid"]))


def check_order(p, cta):
    """Data side: the tile each step reads is the one its group lead loaded."""
    for u in units(p, cta):
        x = make_unit(p, u)
        for s in range(SLOTS):
            if x["len"][s]:
                lo, hi = x["segs"][s]
                first = x["kv_lo"] + x["kt0"][s] * KBN
                assert first <= lo and first + x["len"][s] * KBN >= hi, (u, s, x)
        for rho in range(x["rounds"]):
            loaded = None
            for s in range(SLOTS):
                if not active(x, s, rho):
                    continue
                if lead(x, s, rho):
                    assert loaded is None, ("two leads open", u, rho, s)
                    loaded = x["kt0"][s] + rho
                assert loaded == x["kt0"][s] + rho, ("step reads another tile", u, rho, s, x)
                if last(x, s, rho):
                    loaded = None
            assert loaded is None, ("tile never released", u, rho)


def producer_qk(p, B, cta):
    g, nq = 0, [0] * SLOTS
    for u in units(p, cta):
        x = make_unit(p, u)
        for s in range(SLOTS):
            if x["len"][s] == 0:
                continue
            yield ("wait", B["q_empty"][s], nq[s])
            nq[s] += 1
            B["q_full"][s].arrive()
        for rho in range(x["rounds"]):
            for s in range(SLOTS):
                if lead(x, s, rho):
                    yield ("wait", B["k_empty"][g % KKV], g // KKV)
                    B["k_full"][g % KKV].arrive()
                    g += 1


def producer_v(p, B, cta):
    g = 0
    for u in units(p, cta):
        x = make_unit(p, u)
        for rho in range(x["rounds"]):
            for s in range(SLOTS):
                if lead(x, s, rho):
                    yield ("wait", B["v_empty"][g % KKV], g // KKV)
                    B["v_full"][g % KKV].arrive()
                    g += 1


def qk_issuer(p, B, cta):
    g, nq, used = 0, [0] * SLOTS, [0] * SLOTS
    for u in units(p, cta):
        x = make_unit(p, u)
        for rho in range(x["rounds"]):
            for s in range(SLOTS):
                if not active(x, s, rho):
                    continue
                if rho == 0:
                    nq[s] += 1
                    yield ("wait", B["q_full"][s], nq[s])
                if lead(x, s, rho):
                    yield ("wait", B["k_full"][g % KKV], g // KKV + 1)
                if used[s]:
                    yield ("wait", B["s_free"][s], used[s])
                used[s] += 1
                B["s_full"][s].arrive()
                if rho == x["len"][s] - 1:
                    B["q_empty"][s].arrive()
                if last(x, s, rho):
                    B["k_empty"][g % KKV].arrive()
                    g += 1


def pv_issuer(p, B, cta):
    g, np_, oc = 0, [0] * SLOTS, [0] * SLOTS
    for u in units(p, cta):
        x = make_unit(p, u)
        for rho in range(x["rounds"]):
            for s in range(SLOTS):
                if not active(x, s, rho):
                    continue
                np_[s] += 1
                yield ("wait", B["p_full"][s], np_[s])
                if rho == 0:
                    yield ("wait", B["o_empty"][s], oc[s])
                if lead(x, s, rho):
                    yield ("wait", B["v_full"][g % KKV], g // KKV + 1)
                B["pv_done"][s].arrive()
                B["s_free"][s].arrive()
                if rho == x["len"][s] - 1:
                    B["o_full"][s].arrive()
                    oc[s] += 1
                if last(x, s, rho):
                    B["v_empty"][g % KKV].arrive()
                    g += 1


def softmax(p, B, cta, s, rescale_every=3):
    steps = published = 0
    for u in units(p, cta):
        x = make_unit(p, u)
        for rho in range(x["len"][s]):
            yield ("wait", B["s_full"][s], steps + 1)
            if rho > 0 and rho % rescale_every == 0:  # occasional lazy rescale: pv_done of the previous step
                yield ("wait", B["pv_done"][s], steps)
            steps += 1
            B["p_full"][s].arrive(KBM)
        if x["len"][s] == 0:
            continue
        if published > 0:
            yield ("wait", B["stat_empty"][s], published)
        B["stat_full"][s].arrive(KBM)
        published += 1


def epilogue(p, B, cta):
    par = [0] * SLOTS
    for u in units(p, cta):
        x = make_unit(p, u)
        for s in range(SLOTS):
            if x["len"][s] == 0:
                continue
            yield ("wait", B["o_full"][s], par[s] + 1)
            yield ("wait", B["stat_full"][s], par[s] + 1)
            par[s] += 1
            B["stat_empty"][s].arrive(KBM)
            B["o_empty"][s].arrive(KBM)


def run(p, cta, seed=0):
    mk = lambda name, n, c: [Bar(f"{name}{i}", c) for i in range(n)]  # noqa: E731
    B = dict(q_full=mk("q_full", SLOTS, 1), q_empty=mk("q_empty", SLOTS, 1), k_full=mk("k_full", KKV, 1),
             k_empty=mk("k_empty", KKV, 1), v_full=mk("v_full", KKV, 1), v_empty=mk("v_empty", KKV, 1),
             s_full=mk("s_full", SLOTS, 1), p_full=mk("p_full", SLOTS, KBM), s_free=mk("s_free", SLOTS, 1),
             pv_done=mk("pv_done", SLOTS, 1), o_full=mk("o_full", SLOTS, 1), o_empty=mk("o_empty", SLOTS, KBM),
             stat_full=mk("stat_full", SLOTS, KBM), stat_empty=mk("stat_empty", SLOTS, KBM))
    roles = {"producer_qk": producer_qk(p, B, cta), "producer_v": producer_v(p, B, cta),
             "qk_issuer": qk_issuer(p, B, cta), "pv_issuer": pv_issuer(p, B, cta), "epilogue": epilogue(p, B, cta)}
    for s in range(SLOTS):
        roles[f"softmax{s}"] = softmax(p, B, cta, s)
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
            return {n: (w[1].name, w[2], w[1].phase) for n, w in blocked.items() if w is not None}


def params(N, w, r, h, Bt, grid):
    T, m = N // r, w // r
    n_blocks = -(-T // UNIT)
    return dict(T=T, m=m, h=h, n_blocks=n_blocks, n_units=Bt * h * n_blocks, grid=grid)


def check(N, w, r, h, Bt, grid, seeds=3, max_ctas=None):
    p = params(N, w, r, h, Bt, grid)
    ctas = list(range(min(grid, p["n_units"])))
    if max_ctas:
        ctas = ctas[:max_ctas]
    bad = []
    for c in ctas:
        check_order(p, c)
        for seed in range(seeds):
            try:
                res = run(p, c, seed)
            except ParityHazard as e:
                res = f"PARITY HAZARD {e}"
            if res:
                bad.append((c, seed, res))
                break
    return bad


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=4096)
    ap.add_argument("--w", type=int, default=512)
    ap.add_argument("--r", type=int, default=2)
    ap.add_argument("--h", type=int, default=6)
    ap.add_argument("--B", type=int, default=64)
    ap.add_argument("--grid", type=int, default=148)
    ap.add_argument("--seeds", type=int, default=3)
    a = ap.parse_args()
    bad = check(a.N, a.w, a.r, a.h, a.B, a.grid, a.seeds)
    for b in bad[:3]:
        print(b)
    print(f"{len(bad)} failing CTAs")
