"""CPU checks of the fused multi-branch kernel's host side (csrc/dfa_mb_sm100.cu):
the work-unit schedule `dfa_multibranch_plan` returns (the one the kernel
runs) covers every output row once and gives every (row, branch) pair all the
keys of its segment; and the kernel's mbarrier protocol, dynamic-claim ring
included, is deadlock- and parity-safe (scripts/protocol_model_mb.py)."""
import os
import random
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import protocol_model_mb as pm  # noqa: E402


def spread(h, r):
    return [j % r for j in range(h)]


CASES = [
    (4096, 6, [(512, 1), (1024, 2), (2048, 4), (4096, 8)]),
    (4096, 6, [(256, 2), (512, 2), (1024, 4)]),
    (4096, 6, [(4096, 8), (256, 4), (512, 1)]),
    (4096, 6, [(256, 2), (256, 2)]),
    (4096, 6, [(1024, 4), (2048, 8)]),
    (4096, 6, [(128, 1), (256, 2), (64, 1)]),
    (4096, 6, [(2048, 2), (4096, 4)]),
    (2304, 4, [(256, 1), (512, 2), (1024, 4)]),
    (1000, 4, [(100, 1), (200, 2), (500, 4)]),
    (4096, 4, [(512, 1), (4096, 256)]),
]


def branches(h, spec):
    return [(w, r, spread(h, r)) for w, r in spec]


@pytest.mark.parametrize("n,h,spec", CASES)
def test_schedule_covers_every_row_and_key(n, h, spec):
    brs = branches(h, spec)
    descs, R, gr = pm.plan(n, h, 2, brs)
    pm.check_plan(descs, R, gr, n, h, brs)


def test_schedule_custom_offsets():
    h = 4
    brs = [(256, 1, [0, 0, 0, 0]), (512, 4, [3, 1, 2, 0]), (1024, 8, [7, 5, 5, 2])]
    descs, R, gr = pm.plan(2048, h, 1, brs)
    pm.check_plan(descs, R, gr, 2048, h, brs)


def test_longnet_schedule_shape():
    """LongNet set: 2 offset classes per 128-row query tile (super-units of
    512 rows), 32 steps per super-unit and head, 30 of them with keys."""
    descs, R, gr = pm.plan(4096, 6, 1, branches(6, CASES[0][2]))
    assert (R, gr) == (8, 64)
    assert int(descs["steps"].sum()) == 6 * 8 * 32


@pytest.mark.parametrize("ci", [0, 2, 4, 5, 8])
def test_protocol_deadlock_and_parity_safe(ci):
    n, h, spec = CASES[ci]
    descs, _, _ = pm.plan(n, h, 1, branches(h, spec))
    rnd = random.Random(ci)
    for seed in range(4):
        seq = [rnd.randrange(len(descs)) for _ in range(rnd.randrange(1, 40))]
        assert pm.run_protocol(descs, seq, seed) is None, (ci, seed)


def test_protocol_model_flags_an_early_ring_free():
    """The model is not vacuous: consumers that free their ring slot as soon as
    they take a unit (instead of at their next take) let the producer overwrite
    a descriptor that is still being read -- reported."""
    descs, _, _ = pm.plan(4096, 6, 1, branches(6, CASES[0][2]))
    rnd = random.Random(1)
    pm.EARLY_FREE, pm.KSCHED = True, 2  # a short ring, so the producer's Q-stage gating alone cannot save it
    try:
        with pytest.raises(pm.RingOverwrite):
            for seed in range(8):
                seq = [rnd.randrange(len(descs)) for _ in range(30)]
                pm.run_protocol(descs, seq, seed)
    finally:
        pm.EARLY_FREE, pm.KSCHED = False, 6


def test_plan_rejects_out_of_envelope_sets():
    import paper_2403_09195_b200 as dfa

    with pytest.raises(dfa.UnsupportedError):
        pm.plan(2048, 2, 1, branches(2, [(64, 1), (128, 2), (256, 4), (512, 8), (1024, 16)]))


def _random_sets(seed, count):
    """Random branch sets inside the fused kernel's envelope: intervals with
    r | w, lcm(r) | N, arbitrary per-head offsets."""
    rnd = random.Random(seed)
    out = []
    while len(out) < count:
        n = rnd.choice([512, 768, 1024, 2048, 3072, 4096])
        h = rnd.choice([1, 2, 3, 6])
        nb = rnd.randint(2, 4)
        spec = []
        for _ in range(nb):
            r = rnd.choice([1, 2, 3, 4, 8])
            w = r * rnd.choice([8, 16, 32, 64, 100, 128, 256, 512])
            if w > n:
                continue
            spec.append((w, r, [rnd.randrange(r) for _ in range(h)]))
        if len(spec) < 2:
            continue
        lcm = 1
        for _, r, _ in spec:
            lcm = lcm * r // __import__("math").gcd(lcm, r)
        if n % lcm:
            continue
        out.append((n, h, spec))
    return out


@pytest.mark.parametrize("case", _random_sets(7, 40))
def test_random_sets_schedule(case):
    """Property check of the schedule over random branch sets (sets outside the
    envelope, e.g. > 64 key tiles per unit, must be rejected cleanly)."""
    import paper_2403_09195_b200 as dfa

    n, h, spec = case
    try:
        descs, R, gr = pm.plan(n, h, 1, spec)
    except dfa.UnsupportedError:
        return
    pm.check_plan(descs, R, gr, n, h, spec)
