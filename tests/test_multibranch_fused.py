"""Fused multi-(w, r) kernel (csrc/dfa_mb_sm100.cu): every branch and the LSE
combine in ONE tcgen05 launch, checked against the extension oracle
(oracle/dfa_oracle.c oracle_multibranch_f64: one dense softmax over the
multiset of keys the covering branches select) and against the per-branch
path.  bf16 bar: max|err| <= 2e-2, mean relative <= 1e-2."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BF16_MAX_ABS, BF16_MEAN_REL = 2e-2, 1e-2


def _torch():
    import torch

    return torch


def _inputs(B, n, h, seed):
    torch = _torch()
    g = torch.Generator(device="cuda").manual_seed(seed)
    return tuple(torch.randn((B, n, h, 64), device="cuda", generator=g, dtype=torch.bfloat16) for _ in range(3))


def _full(dfa, h, branches):
    out = []
    for br in branches:
        w, r = br[0], br[1]
        offs = list(br[2]) if len(br) > 2 else dfa.AttentionConfig.spread_offsets(h, r)
        out.append((w, r, offs))
    return out


SETS = [
    [(512, 1), (1024, 2), (2048, 4), (4096, 8)],      # LongNet geometric set
    [(256, 2), (512, 2), (1024, 4)],
    [(4096, 8), (256, 4), (512, 1)],                  # sparse first branch
    [(256, 2), (256, 2)],                             # duplicate branch (weights 1/2)
    [(1024, 4), (2048, 8)],                           # no r = 1: rows / tiles no branch selects
    [(128, 1), (256, 2), (64, 1)],                    # segments shorter than a query tile's span
    [(2048, 2), (4096, 4)],
]


@pytest.mark.timeout(300)
@pytest.mark.parametrize("si", range(len(SETS)))
def test_fused_vs_extension_oracle(dfa, port, cuda, si):
    torch = _torch()
    branches = SETS[si]
    B, n, h = 2, 4096, 6
    q, k, v = _inputs(B, n, h, 100 + si)
    cfg = dfa.AttentionConfig(n, branches[0][0], branches[0][1], h, 64,
                              dfa.AttentionConfig.spread_offsets(h, branches[0][1]))
    L = torch.full((B, h, n), float("nan"), device="cuda")
    o = torch.full((B, n, h, 64), float("nan"), device="cuda", dtype=torch.bfloat16)
    dfa.dfa_forward_multibranch(q, k, v, cfg, branches, out=o, lse=L)
    assert dfa.last_launch_count() == 1, "fused single-kernel path not taken"
    torch.cuda.synchronize()
    want, want_lse = port.multibranch_batched(*(x.double().cpu().numpy() for x in (q, k, v)),
                                              _full(dfa, h, branches))
    got = o.double().cpu().numpy()
    assert np.isfinite(got).all()
    err = np.abs(got - want)
    mx, rel = float(err.max()), float(err.sum() / np.abs(want).sum())
    assert mx <= BF16_MAX_ABS and rel <= BF16_MEAN_REL, (branches, mx, rel)
    Lg = L.cpu().numpy()
    fin = np.isfinite(want_lse)
    assert np.array_equal(np.isfinite(Lg), fin)
    assert np.abs(Lg[fin] - want_lse[fin]).max() <= 2e-2
    # rows no branch selects: exact zeros (the buffer was NaN-poisoned)
    unsel = ~fin.transpose(0, 2, 1)  # [B, N, h]
    assert (got[unsel] == 0).all()


@pytest.mark.timeout(300)
def test_fused_custom_offsets(dfa, port, cuda):
    """Per-branch head offsets that are not j mod r (any class mapping)."""
    torch = _torch()
    B, n, h = 1, 2048, 4
    branches = [(256, 1, [0, 0, 0, 0]), (512, 4, [3, 1, 2, 0]), (1024, 8, [7, 5, 5, 2])]
    q, k, v = _inputs(B, n, h, 5)
    cfg = dfa.AttentionConfig(n, 256, 1, h, 64, [0] * h)
    L = torch.empty((B, h, n), device="cuda")
    o = dfa.dfa_forward_multibranch(q, k, v, cfg, branches, lse=L)
    assert dfa.last_launch_count() == 1
    torch.cuda.synchronize()
    want, want_lse = port.multibranch_batched(*(x.double().cpu().numpy() for x in (q, k, v)), branches)
    err = np.abs(o.double().cpu().numpy() - want)
    assert err.max() <= BF16_MAX_ABS and err.sum() / np.abs(want).sum() <= BF16_MEAN_REL


@pytest.mark.timeout(300)
@pytest.mark.parametrize("si", [0, 2, 4])
def test_fused_vs_per_branch_full_batch(dfa, cuda, si):
    """B = 64, h = 6 (the bench batch): fused kernel vs the per-branch launches
    (epilogue merge); bitwise-deterministic across runs."""
    torch = _torch()
    from paper_2403_09195_b200 import _lib, multibranch_mode

    branches = SETS[si]
    B, n, h = 64, 4096, 6
    q, k, v = _inputs(B, n, h, 7 + si)
    cfg = dfa.AttentionConfig(n, 512, 1, h, 64, [0] * h)
    a = dfa.dfa_forward_multibranch(q, k, v, cfg, branches)
    assert dfa.last_launch_count() == 1
    a2 = dfa.dfa_forward_multibranch(q, k, v, cfg, branches)
    with multibranch_mode(_lib.DFA_MB_PER_BRANCH):
        b = dfa.dfa_forward_multibranch(q, k, v, cfg, branches)
        assert dfa.last_launch_count() == len(branches)
    torch.cuda.synchronize()
    assert torch.equal(a, a2)
    err = (a.float() - b.float()).abs()
    assert err.max().item() <= BF16_MAX_ABS
    assert (err.sum() / b.float().abs().sum()).item() <= BF16_MEAN_REL


def test_fused_outside_envelope_falls_back(dfa, cuda):
    """Five distinct intervals (> 4 tensor-map slots): per-branch launches."""
    torch = _torch()
    branches = [(64, 1), (128, 2), (256, 4), (512, 8), (1024, 16)]
    q, k, v = _inputs(1, 2048, 2, 3)
    cfg = dfa.AttentionConfig(2048, 64, 1, 2, 64, [0, 0])
    a = dfa.dfa_forward_multibranch(q, k, v, cfg, branches)
    assert dfa.last_launch_count() == len(branches)
    torch.cuda.synchronize()
    assert torch.isfinite(a.float()).all()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("n,branches", [
    (2304, [(256, 1), (512, 2), (1024, 4)]),   # tail super-unit, tail segments
    (1000, [(100, 1), (200, 2), (500, 4)]),    # short segments, N not a multiple of the tile span
    (4096, [(512, 1), (4096, 256)]),            # R = 256 offset classes
])
def test_fused_tails_vs_oracle(dfa, port, cuda, n, branches):
    torch = _torch()
    B, h = 3, 4
    q, k, v = _inputs(B, n, h, n)
    cfg = dfa.AttentionConfig(n, branches[0][0], branches[0][1], h, 64,
                              dfa.AttentionConfig.spread_offsets(h, branches[0][1]))
    L = torch.empty((B, h, n), device="cuda")
    o = torch.full((B, n, h, 64), float("nan"), device="cuda", dtype=torch.bfloat16)
    dfa.dfa_forward_multibranch(q, k, v, cfg, branches, out=o, lse=L)
    assert dfa.last_launch_count() == 1
    torch.cuda.synchronize()
    want, want_lse = port.multibranch_batched(*(x.double().cpu().numpy() for x in (q, k, v)),
                                              _full(dfa, h, branches))
    got = o.double().cpu().numpy()
    err = np.abs(got - want)
    assert np.isfinite(got).all()
    assert err.max() <= BF16_MAX_ABS and err.sum() / np.abs(want).sum() <= BF16_MEAN_REL
    fin = np.isfinite(want_lse)
    assert np.array_equal(np.isfinite(L.cpu().numpy()), fin)


def test_fused_small_batch_and_graph_replay(dfa, cuda):
    """B = 1 (fewer units than SMs) and CUDA-graph replays of the fused launch
    (the work counters re-arm at the end of every launch)."""
    torch = _torch()
    branches = SETS[0]
    q, k, v = _inputs(1, 4096, 6, 11)
    cfg = dfa.AttentionConfig(4096, 512, 1, 6, 64, [0] * 6)
    s = torch.cuda.Stream()
    o = torch.empty_like(q)
    with torch.cuda.stream(s):
        ref = dfa.dfa_forward_multibranch(q, k, v, cfg, branches, stream=s)  # uploads the schedule for s
        assert dfa.last_launch_count() == 1
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        dfa.dfa_forward_multibranch(q, k, v, cfg, branches, out=o, stream=s)
    assert dfa.last_launch_count() == 1, "fused kernel not captured"
    for _ in range(3):
        o.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(o, ref)


def test_fused_plan_cache_eviction(dfa, cuda):
    """More branch sets than the schedule cache holds (16): evicted plans are
    rebuilt on their next use and results stay identical."""
    torch = _torch()
    q, k, v = _inputs(1, 1024, 2, 21)
    cfg = dfa.AttentionConfig(1024, 128, 1, 2, 64, [0, 0])
    first = [(128, 1), (256, 2)]
    a = dfa.dfa_forward_multibranch(q, k, v, cfg, first)
    others = [[(64 * w, 1), (512, 2)] for w in range(1, 17)] + [[(64 * w, 1), (1024, 4)] for w in range(1, 5)]
    for br in others:  # 20 further distinct sets
        dfa.dfa_forward_multibranch(q, k, v, cfg, br)
        assert dfa.last_launch_count() == 1
    b = dfa.dfa_forward_multibranch(q, k, v, cfg, first)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("branches,fused", [
    ([(4096, 1), (2048, 1)], True),              # 48 key tiles per unit: still one launch
    ([(4096, 1), (4096, 1), (4096, 2)], False),  # 80 > 64 key tiles per unit: per-branch launches
])
def test_long_segment_sets(dfa, cuda, branches, fused):
    torch = _torch()
    from paper_2403_09195_b200 import _lib, multibranch_mode

    q, k, v = _inputs(4, 4096, 6, 17)
    cfg = dfa.AttentionConfig(4096, 4096, 1, 6, 64, [0] * 6)
    a = dfa.dfa_forward_multibranch(q, k, v, cfg, branches)
    assert dfa.last_launch_count() == (1 if fused else len(branches))
    with multibranch_mode(_lib.DFA_MB_PER_BRANCH):
        b = dfa.dfa_forward_multibranch(q, k, v, cfg, branches)
    torch.cuda.synchronize()
    err = (a.float() - b.float()).abs()
    assert err.max().item() <= BF16_MAX_ABS
    assert (err.sum() / b.float().abs().sum()).item() <= BF16_MEAN_REL


def test_first_call_under_capture_takes_per_branch_path(dfa, cuda):
    """A branch set seen for the first time inside a CUDA-graph capture cannot
    upload its schedule: that call takes the per-branch launches (still
    captured, still correct)."""
    torch = _torch()
    branches = [(512, 1), (1024, 2), (2048, 4)]
    q, k, v = _inputs(2, 4096, 6, 23)
    cfg = dfa.AttentionConfig(4096, 512, 1, 6, 64, [0] * 6)
    ref = dfa.dfa_forward_multibranch(q, k, v, cfg, branches)  # default stream: its own plan
    s = torch.cuda.Stream()
    o = torch.empty_like(q)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        dfa.dfa_forward_multibranch(q, k, v, cfg, branches, out=o, stream=s)
    assert dfa.last_launch_count() == len(branches)
    g.replay()
    torch.cuda.synchronize()
    err = (o.float() - ref.float()).abs()
    assert err.max().item() <= BF16_MAX_ABS


def _random_sets(seed, count):
    """Random branch sets (r | w, lcm(r) | N, random per-head offsets) -- the
    same generator as tests/test_mb_plan.py's schedule property test, smaller
    sizes so the f64 oracle stays fast."""
    import math
    import random

    rnd = random.Random(seed)
    out = []
    while len(out) < count:
        n = rnd.choice([512, 768, 1024, 2048])
        h = rnd.choice([1, 2, 3])
        spec = []
        for _ in range(rnd.randint(2, 4)):
            r = rnd.choice([1, 2, 3, 4, 8])
            w = r * rnd.choice([8, 16, 32, 64, 100, 128, 256])
            if w <= n:
                spec.append((w, r, [rnd.randrange(r) for _ in range(h)]))
        if len(spec) >= 2 and n % math.lcm(*(r for _, r, _ in spec)) == 0:
            out.append((n, h, spec))
    return out


@pytest.mark.timeout(300)
@pytest.mark.parametrize("case", _random_sets(11, 10))
def test_random_sets_vs_oracle(dfa, port, cuda, case):
    torch = _torch()
    n, h, branches = case
    B = 2
    q, k, v = _inputs(B, n, h, n + h)
    w0, r0, off0 = branches[0]
    cfg = dfa.AttentionConfig(n, w0, r0, h, 64, off0)
    L = torch.full((B, h, n), float("nan"), device="cuda")
    o = torch.full((B, n, h, 64), float("nan"), device="cuda", dtype=torch.bfloat16)
    dfa.dfa_forward_multibranch(q, k, v, cfg, branches, out=o, lse=L)
    assert dfa.last_launch_count() == 1, "all these sets are inside the fused kernel's envelope"
    torch.cuda.synchronize()
    want, want_lse = port.multibranch_batched(*(x.double().cpu().numpy() for x in (q, k, v)), branches)
    got = o.double().cpu().numpy()
    assert np.isfinite(got).all()
    err = np.abs(got - want)
    assert err.max() <= BF16_MAX_ABS and err.sum() / max(np.abs(want).sum(), 1e-30) <= BF16_MEAN_REL, (case, err.max())
    fin = np.isfinite(want_lse)
    Lg = L.cpu().numpy()
    assert np.array_equal(np.isfinite(Lg), fin)
    assert np.abs(Lg[fin] - want_lse[fin]).max() <= 2e-2


@pytest.mark.timeout(300)
def test_fused_repeatable_back_to_back(dfa, cuda):
    """Stress: 25 back-to-back fused launches (dynamic unit claiming, counters
    re-armed by the last CTA of each launch, PDL overlap of consecutive
    launches) on two alternating branch sets give bitwise identical outputs."""
    torch = _torch()
    q, k, v = _inputs(16, 4096, 6, 29)
    cfg = dfa.AttentionConfig(4096, 512, 1, 6, 64, [0] * 6)
    sets = [SETS[0], SETS[1]]
    refs = [dfa.dfa_forward_multibranch(q, k, v, cfg, br) for br in sets]
    outs = [torch.empty_like(q) for _ in sets]
    for i in range(25):
        j = i % 2
        dfa.dfa_forward_multibranch(q, k, v, cfg, sets[j], out=outs[j])
        assert dfa.last_launch_count() == 1
        if i >= 23:
            torch.cuda.synchronize()
            assert torch.equal(outs[j], refs[j])
