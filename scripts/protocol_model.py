#!/usr/bin/env python3
"""Executable model of dfa_sm100_kernel's mbarrier protocol (one CTA).

Each warp role is a Python generator mirroring the kernel's loops; it yields
('wait', barrier, parity) and performs arrivals / commits directly (async TMA
and MMA completions are modelled as immediate).  A round-robin scheduler runs
the roles; if no role can make progress before all finish, the protocol
deadlocks and the blocked waits are printed.

    python scripts/protocol_model.py --N 4096 --w 256 --r 2 --h 6 --B 64 --grid 148 --cta 10
"""
import argparse
import math

KBM = 128
KBN = 128
KSB = 3   # S buffers
KKV = 3   # K / V ring depth
KQ = 2


class ParityHazard(AssertionError):
    pass


class Bar:
    def __init__(self, name, count):
        self.name, self.count, self.pending, self.phase = name, count, count, 0

    def arrive(self, n=1):
        self.pending -= n
        assert self.pending >= 0, f"over-arrival on {self.name}"
        if self.pending == 0:
            self.phase += 1
            self.pending = self.count

    def done(self, need):
        """Wait for `need` completed phases, the way the kernel does it:
        try_wait.parity((need - 1) & 1) succeeds iff the current (incomplete)
        phase has the other parity.  That is only correct while the completed
        count is need - 1 or need; anything else is a parity hazard (early
        return or a wait that can never succeed)."""
        if need <= 0:
            return True
        if not (need - 1 <= self.phase <= need):
            raise ParityHazard(f"{self.name}: waiting for {need} completions, barrier has {self.phase}")
        return (self.phase & 1) != ((need - 1) & 1)


def make_unit(p, u):
    j, bp = u % p["h"], u // p["h"]  # head-major unit order (DFA_HEAD_MAJOR)
    pair, b = bp % p["n_pairs"], bp // p["n_pairs"]
    unit = p.get("unit_rows", 2 * KBM)
    t0 = pair * unit
    lo, hi = [], []
    for s in range(2):
        r0 = t0 + s * KBM
        r1 = r0 if (s == 1 and unit == KBM) else min(r0 + KBM, p["T"])  # half units: slot B empty
        if r0 < r1:
            lo.append((r0 // p["m"]) * p["m"])
            hi.append(min(((r1 - 1) // p["m"] + 1) * p["m"], p["T"]))
        else:
            lo.append(-1)
            hi.append(-1)
    kv_lo = lo[0]
    kv_hi = max(hi[0], hi[1]) if hi[1] >= 0 else hi[0]
    n_kv = -(-(kv_hi - kv_lo) // KBN)
    kt = [((lo[0] - kv_lo) // KBN, -(-(hi[0] - kv_lo) // KBN))]
    kt.append((0, 0) if lo[1] < 0 else ((lo[1] - kv_lo) // KBN, -(-(hi[1] - kv_lo) // KBN)))
    return dict(b=b, j=j, t0=t0, kv_lo=kv_lo, n_kv=n_kv, kt=kt)


def uses(x, s, kt):
    return x["kt"][s][0] <= kt < x["kt"][s][1]


def steps_of(x):
    return sum(b - a for a, b in x["kt"])


def step_in_unit(x, kt, s):
    cc = lambda kt, lo, hi: min(max(kt, lo), hi) - lo  # noqa: E731
    return cc(kt, *x["kt"][0]) + cc(kt, *x["kt"][1]) + (1 if s == 1 and uses(x, 0, kt) else 0)


def units(p, cta):
    return list(range(cta, p["n_units"], p["grid"]))


def producer_qk(p, B, cta):
    g = 0
    for i, u in enumerate(units(p, cta)):
        x = make_unit(p, u)
        qs = i % KQ
        yield ("wait", B["q_empty"][qs], i // KQ)
        B["q_full"][qs].arrive()  # TMA complete_tx modelled as immediate
        for kt in range(x["n_kv"]):
            st = g % KKV
            yield ("wait", B["k_empty"][st], g // KKV)
            B["k_full"][st].arrive()
            g += 1


def producer_v(p, B, cta):
    g = 0
    for u in units(p, cta):
        x = make_unit(p, u)
        for kt in range(x["n_kv"]):
            st = g % KKV
            yield ("wait", B["v_empty"][st], g // KKV)
            B["v_full"][st].arrive()
            g += 1


def step_list(p, cta):
    """(i, unit, kt, s, g) in the MMA's order."""
    out, g = [], 0
    for i, u in enumerate(units(p, cta)):
        x = make_unit(p, u)
        for kt in range(x["n_kv"]):
            for s in range(2):
                if uses(x, s, kt):
                    out.append((i, x, kt, s, g))
            g += 1
    return out


def qk_issuer(p, B, cta):
    """warp 1: Q K^T for step k into S buffer k % 3 once P V of step k - 3 completed."""
    steps = 0
    g = 0
    for i, u in enumerate(units(p, cta)):
        x = make_unit(p, u)
        qs = i & 1
        yield ("wait", B["q_full"][qs], (i >> 1) + 1)
        for kt in range(x["n_kv"]):
            yield ("wait", B["k_full"][g % KKV], g // KKV + 1)
            for s in range(2):
                if not uses(x, s, kt):
                    continue
                b = steps % KSB
                if steps >= KSB:
                    yield ("wait", B["s_free"][b], steps // KSB)
                B["s_full"][s][b].arrive()
                steps += 1
            B["k_empty"][g % KKV].arrive()
            g += 1
        B["q_empty"][qs].arrive()


def pv_issuer(p, B, cta):
    """warp 2: P V for step k after P(k); frees S buffer k % 3 (s_free)."""
    steps = 0
    g = 0
    oc = [0, 0]
    for i, u in enumerate(units(p, cta)):
        x = make_unit(p, u)
        for kt in range(x["n_kv"]):
            have_v = False
            for s in range(2):
                if not uses(x, s, kt):
                    continue
                b = steps % KSB
                yield ("wait", B["p_full"][b], steps // KSB + 1)
                if kt == x["kt"][s][0]:
                    yield ("wait", B["o_empty"][s], oc[s])
                if not have_v:
                    yield ("wait", B["v_full"][g % KKV], g // KKV + 1)
                    have_v = True
                B["pv_done"][s].arrive()
                B["s_free"][b].arrive()
                if kt == x["kt"][s][1] - 1:
                    B["o_full"][s].arrive()
                    oc[s] += 1
                steps += 1
            B["v_empty"][g % KKV].arrive()
            g += 1


def softmax(p, B, cta, s):
    use_par = [0, 0, 0]
    pvc = steps_done = 0
    k_base = 0
    published = 0  # units whose stats this slot handed to the epilogue
    for i, u in enumerate(units(p, cta)):
        x = make_unit(p, u)
        lo, hi = x["kt"][s]
        k_unit = k_base
        k_base += steps_of(x)
        if lo == hi:
            continue
        for kt in range(lo, hi):
            b = (k_unit + step_in_unit(x, kt, s)) % KSB
            yield ("wait", B["s_full"][s][b], use_par[b] + 1)
            use_par[b] += 1
            if steps_done > 0:
                yield ("wait", B["pv_done"][s], pvc + 1)
                pvc += 1
            steps_done += 1
            B["p_full"][b].arrive(KBM)
        # stats go to buffer (published & 1); publish only once the epilogue
        # consumed the previous unit's, so stat_full is never 2 phases ahead
        if published > 0:
            yield ("wait", B["stat_empty"][s], published)
        B["stat_full"][s].arrive(KBM)
        published += 1


def epilogue(p, B, cta):
    par = [0, 0]
    for i, u in enumerate(units(p, cta)):
        x = make_unit(p, u)
        for s in range(2):
            if x["kt"][s][0] == x["kt"][s][1]:
                continue
            yield ("wait", B["o_full"][s], par[s] + 1)
            yield ("wait", B["stat_full"][s], par[s] + 1)
            par[s] += 1
            B["stat_empty"][s].arrive(KBM)
            B["o_empty"][s].arrive(KBM)


def run(p, cta, seed=0):
    B = dict(q_full=[Bar(f"q_full{i}", 1) for i in range(KQ)], q_empty=[Bar(f"q_empty{i}", 1) for i in range(KQ)],
             k_full=[Bar(f"k_full{i}", 1) for i in range(KKV)], k_empty=[Bar(f"k_empty{i}", 1) for i in range(KKV)],
             v_full=[Bar(f"v_full{i}", 1) for i in range(KKV)], v_empty=[Bar(f"v_empty{i}", 1) for i in range(KKV)],
             s_full=[[Bar(f"s_full{s}{b}", 1) for b in range(KSB)] for s in range(2)],
             p_full=[Bar(f"p_full{b}", KBM) for b in range(KSB)],
             s_free=[Bar(f"s_free{b}", 1) for b in range(KSB)], pv_done=[Bar(f"pv_done{s}", 1) for s in range(2)],
             o_full=[Bar(f"o_full{s}", 1) for s in range(2)], o_empty=[Bar(f"o_empty{s}", KBM) for s in range(2)],
             stat_full=[Bar(f"stat_full{s}", KBM) for s in range(2)],
             stat_empty=[Bar(f"stat_empty{s}", KBM) for s in range(2)])
    roles = {"producer_qk": producer_qk(p, B, cta), "producer_v": producer_v(p, B, cta), "qk_issuer": qk_issuer(p, B, cta), "pv_issuer": pv_issuer(p, B, cta),
             "softmax_A": softmax(p, B, cta, 0), "softmax_B": softmax(p, B, cta, 1), "epilogue": epilogue(p, B, cta)}
    import random

    rnd = random.Random(seed)
    blocked = {}
    for name, gen in roles.items():
        blocked[name] = next(gen, None)
    names = list(roles)
    while True:
        progress = False
        if seed:
            rnd.shuffle(names)
        for name in names:
            gen = roles[name]
            w = blocked[name]
            while w is not None and w[1].done(w[2]):
                w = next(gen, None)
                progress = True
            blocked[name] = w
        if all(w is None for w in blocked.values()):
            return None
        if not progress:
            return {n: (w[1].name, w[2], w[1].phase) for n, w in blocked.items() if w is not None}


def params(N, w, r, h, Bt, grid, sms=148):
    """Mirror of launch_sm100's unit geometry (half units when the grid is small)."""
    T, m = N // r, w // r
    unit = 2 * KBM
    n_pairs = -(-T // unit)
    if Bt * h * -(-T // KBM) <= sms:
        unit = KBM
        n_pairs = -(-T // unit)
    return dict(T=T, m=m, h=h, n_pairs=n_pairs, n_units=Bt * h * n_pairs, grid=grid, unit_rows=unit)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=4096)
    ap.add_argument("--w", type=int, default=256)
    ap.add_argument("--r", type=int, default=2)
    ap.add_argument("--h", type=int, default=6)
    ap.add_argument("--B", type=int, default=64)
    ap.add_argument("--grid", type=int, default=148)
    ap.add_argument("--cta", type=int, default=-1)
    ap.add_argument("--seeds", type=int, default=4)
    a = ap.parse_args()
    p = params(a.N, a.w, a.r, a.h, a.B, a.grid)
    ctas = [a.cta] if a.cta >= 0 else range(min(a.grid, p["n_units"]))
    bad = 0
    for c in ctas:
        for seed in range(a.seeds):
            try:
                res = run(p, c, seed)
            except ParityHazard as e:
                res = f"PARITY HAZARD {e}"
            if res:
                bad += 1
                if bad <= 3:
                    print(f"CTA {c} seed {seed}: {res}")
                break
    print(f"{bad} failing CTAs of {len(list(ctas))}")
