"""Pin the oracle before trusting it (CPU only).

The C restatement (oracle/dfa_oracle.c) must be BIT-IDENTICAL to the
unmodified reference (oracle/_ref, built from /root/reference), and both must
reproduce the reference's own known answers (test_attention.cpp) and
acceptance gates 1, 3, 4 (acceptance.cpp).
"""
import numpy as np
import pytest

from conftest import rand

# (N, w, r) grid: exact division, tails (w !| N), r !| w, single rows, collapse.
GRID = [
    (8, 4, 2), (16, 4, 2), (16, 8, 4), (10, 4, 2), (33, 7, 3), (12, 12, 1), (100, 30, 4),
    (64, 16, 2), (5, 5, 5), (7, 3, 3), (1, 1, 1), (40, 40, 8), (257, 64, 4),
]


@pytest.mark.parametrize("n,w,r", GRID)
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_port_bit_identical_to_reference(port, ref, n, w, r, dtype):
    for g in range(r):
        for tiled, tile in ((False, 1), (True, 1), (True, 3), (True, 64)):
            seed = hash((n, w, r, g, tile)) % 2**31
            q, k = rand((n, 8), seed, dtype), rand((n, 8), seed + 1, dtype)
            v = rand((n, 5), seed + 2, dtype)
            a = port.dilated_attention(q, k, v, w, r, g, tiled=tiled, tile=tile)
            b = ref.dilated_attention(q, k, v, w, r, g, tiled=tiled, tile=tile)
            assert a.tobytes() == b.tobytes(), (n, w, r, g, tiled, tile)


def test_port_bit_identical_headline_f32(port, ref):
    """Config 1: N=4096, w=512, r=2, d=64, gamma=0, fp32."""
    q, k, v = (rand((4096, 64), s, np.float32) for s in (901, 902, 903))
    a = port.dilated_attention(q, k, v, 512, 2, 0)
    b = ref.dilated_attention(q, k, v, 512, 2, 0)
    assert a.tobytes() == b.tobytes()


def test_unscaled_scores_mode(port, ref):
    q, k, v = (rand((16, 4), s) for s in (1, 2, 3))
    a = port.dilated_attention(q, k, v, 8, 2, 1, scale=False)
    b = ref.dilated_attention(q, k, v, 8, 2, 1, scale=False)
    assert a.tobytes() == b.tobytes()


def test_workers_do_not_change_bits(ref):
    """acceptance gate 8 / test_attention.cpp:360-369."""
    q, k, v = (rand((64, 8), s) for s in (604, 605, 606))
    assert ref.dilated_attention(q, k, v, 16, 2, 1, workers=1).tobytes() == \
        ref.dilated_attention(q, k, v, 16, 2, 1, workers=4).tobytes()


def test_masked_oracle_gate1(port, ref):
    """acceptance.cpp:57-84: (N,w,r) in {8,16,32}x{2,4,8}x{1,2,4}, all gamma, d=8, tol 1e-10."""
    worst, configs = 0.0, 0
    for n in (8, 16, 32):
        for w in (2, 4, 8):
            if w > n or n % w:
                continue
            for r in (1, 2, 4):
                if r > w or w % r:
                    continue
                for g in range(r):
                    q, k, v = (rand((n, 8), 10 * configs + s) for s in range(3))
                    d1 = port.dilated_attention(q, k, v, w, r, g)
                    worst = max(worst, np.abs(d1 - port.masked_dense(q, k, v, w, r, g)).max())
                    worst = max(worst, np.abs(d1 - ref.masked_dense(q, k, v, w, r, g)).max())
                    configs += 1
    assert configs >= 27
    assert worst <= 1e-10


def test_collapse_gate3(port, ref):
    """acceptance.cpp:119-138: w = N, r = 1 equals dense attention, f32 <= 1e-6."""
    for seed in range(20):
        n = 8 + seed * 3
        q, k, v = (rand((n, 8), 300 + seed * 3 + s, np.float32) for s in range(3))
        got = port.dilated_attention(q, k, v, n, 1, 0)
        assert np.abs(got - ref.naive_attention(q, k, v)).max() <= 1e-6


# --------------------------------------------------------- index goldens
def test_segment_view_goldens(port, ref, dfa):
    """test_attention.cpp:148-179."""
    for impl in (port.segment_view, ref.segment_view,
                 lambda *a: dfa.make_segment_view(*a).row_indices):
        assert impl(8, 4, 2, 1, 0) == [4, 6]
        assert impl(8, 4, 1, 0, 0) == [0, 1, 2, 3]
        assert impl(10, 4, 2, 2, 1) == [9]


def test_segment_view_random_walk(port, ref, dfa):
    """test_attention.cpp:181-201: stride r, inside the segment, m = ceil((rows-g)/r)."""
    rng = np.random.default_rng(304)
    for _ in range(200):
        n = int(rng.integers(4, 65))
        w = int(rng.integers(1, n + 1))
        r = int(rng.integers(1, w + 1))
        i = int(rng.integers(0, (n + w - 1) // w))
        g = int(rng.integers(0, r))
        a = ref.segment_view(n, w, r, i, g)
        assert port.segment_view(n, w, r, i, g) == a
        assert dfa.make_segment_view(n, w, r, i, g).row_indices == a
        lo, hi = i * w, min(i * w + w, n)
        assert all(lo <= x < hi for x in a)
        assert all(b - a_ == r for a_, b in zip(a, a[1:]))
        rows = hi - lo
        assert len(a) == (0 if g >= rows else (rows - g + r - 1) // r)


def test_segment_view_bounds(port, ref, dfa):
    """test_attention.cpp:203-210."""
    from oracle.oracle import OracleError

    for args in ((8, 4, 2, 2, 0), (8, 4, 2, -1, 0), (8, 4, 2, 0, 2)):
        with pytest.raises(OracleError):
            ref.segment_view(*args)
        with pytest.raises(OracleError):
            port.segment_view(*args)
        with pytest.raises(dfa.OutOfRange) as e:
            dfa.make_segment_view(*args)
        with pytest.raises(OracleError) as e2:
            ref.segment_view(*args)
        assert str(e.value) in str(e2.value)


def test_slice_scatter_partition():
    """verify.hpp:143-155: the r offset classes partition the rows exactly."""
    from paper_2403_09195_b200 import make_segment_view

    for n, w, r in ((12, 12, 3), (50, 8, 4), (4096, 512, 2)):
        seen = np.zeros(n, dtype=int)
        for i in range((n + w - 1) // w):
            for g in range(r):
                seen[make_segment_view(n, w, r, i, g).row_indices] += 1
        assert (seen == 1).all()


# ---------------------------------------------------------- flop goldens
def test_flop_goldens(port, ref, dfa):
    """test_attention.cpp:444-482 and acceptance gate 4."""
    assert ref.flop_count(4096, 512, 2, 1, 64, [0])[:3] == (2147483648, 67108864, 32.0)
    assert ref.flop_count(4096, 512, 2, 1, 64, [0])[3] == "4096,512,2,1,64,2147483648,67108864,32"
    assert ref.flop_count(4096, 2048, 2, 1, 64, [0])[2] == 8.0
    assert ref.flop_count(64, 64, 1, 1, 4, [0])[2] == 1.0
    cfg = dfa.AttentionConfig(4096, 512, 2, 1, 64, [0])
    fc = dfa.flop_count(cfg)
    assert (fc.dense_mults, fc.dilated_mults, fc.ratio) == (2147483648, 67108864, 32.0)
    assert dfa.flop_csv_header() == "N,w,r,h,d,dense_mults,dilated_mults,ratio"
    assert dfa.flop_csv_row(cfg, fc) == "4096,512,2,1,64,2147483648,67108864,32"
    for n, w, r in ((4096, 512, 2), (1024, 512, 2), (64, 16, 2), (256, 64, 4), (128, 128, 1), (2048, 256, 4),
                    (32, 8, 2)):
        want = n * r * r / w
        assert ref.flop_count(n, w, r, 1, 64, [0])[2] == want
        assert port.flop_count(n, w, r, 1, 64, [0])[2] == want
        assert dfa.flop_count(dfa.AttentionConfig(n, w, r, 1, 64, [0])).ratio == want
    for n, w, r, h in ((4096, 512, 2, 6), (100, 30, 4, 3), (10, 4, 2, 2)):
        offs = dfa.AttentionConfig.spread_offsets(h, r)
        a = ref.flop_count(n, w, r, h, 64, offs)[:3]
        assert port.flop_count(n, w, r, h, 64, offs) == a
        got = dfa.flop_count(dfa.AttentionConfig(n, w, r, h, 64, offs))
        assert (got.dense_mults, got.dilated_mults, got.ratio) == a


def test_flop_ratio_monotone(dfa):
    """test_attention.cpp:462-475."""
    prev = 0.0
    for r in (1, 2, 4, 8, 16):
        x = dfa.flop_count(dfa.AttentionConfig(64, 16, r, 1, 4, [0])).ratio
        assert x > prev
        prev = x
    prev = float("inf")
    for w in (4, 8, 16, 32, 64):
        x = dfa.flop_count(dfa.AttentionConfig(64, w, 2, 1, 4, [0])).ratio
        assert x < prev
        prev = x


# ------------------------------------------------------- validation rules
VALIDATE_CASES = [
    # (n, w, r, h, d, offsets, tiled, tile, full)
    (8, 9, 1, 1, 4, [0], 0, 1, 0),     # w > N
    (8, 4, 5, 1, 4, [0], 0, 1, 0),     # r > w
    (0, 4, 2, 1, 4, [0], 0, 1, 0),     # N = 0
    (8, 4, 2, 1, 4, [2], 0, 1, 0),     # offset outside [0, r)
    (8, 4, 2, 1, 4, [-1], 0, 1, 0),
    (8, 4, 2, 1, 0, [0], 0, 1, 0),     # d = 0
    (8, 4, 2, 1, 4, [0], 1, 0, 0),     # tiled with tile 0
    (8, 4, 2, 2, 4, [0, 0], 0, 1, 1),  # coverage violation
    (8, 4, 2, 2, 4, [0, 1], 0, 1, 1),  # ok
    (8, 4, 2, 2, 4, [0, 0], 0, 1, 0),  # ok without coverage
    (16, 8, 4, 3, 4, [0, 1, 2], 0, 1, 1),  # h < r
    (4096, 512, 2, 6, 64, [0, 1, 0, 1, 0, 1], 0, 1, 1),
]


@pytest.mark.parametrize("case", VALIDATE_CASES)
def test_validate_matches_reference(ref, port, dfa, case):
    n, w, r, h, d, offs, tiled, tile, full = case
    st_ref, msg_ref = ref.validate(n, w, r, h, d, offs, tiled, tile, full)
    assert port.validate(n, w, r, h, d, offs, tiled, tile, full) == st_ref
    cfg = dfa.AttentionConfig(n, w, r, h, d, list(offs), "tiled" if tiled else "naive", tile)
    if st_ref == 0:
        cfg.validate(bool(full))
    else:
        with pytest.raises(dfa.ConfigError) as e:
            cfg.validate(bool(full))
        assert str(e.value) == msg_ref


def test_offset_count_mismatch(ref, dfa):
    st, msg = ref.validate(8, 4, 2, 1, 4, [0, 0])
    assert st == 1
    with pytest.raises(dfa.ConfigError) as e:
        dfa.AttentionConfig(8, 4, 2, 1, 4, [0, 0]).validate()
    assert str(e.value) == msg


# ------------------------------------------------- extension oracles (LSE)
def test_multibranch_single_branch_is_dilated(port):
    """The LSE-combine oracle reduces to dilated_attention with one branch."""
    for n, w, r, g in ((64, 16, 2, 1), (100, 30, 4, 3), (4096, 512, 2, 0)):
        q, k, v = (rand((n, 16), s) for s in (7, 8, 9))
        mb, _ = port.multibranch(q, k, v, [(w, r, g)])
        assert np.abs(mb - port.dilated_attention(q, k, v, w, r, g)).max() <= 1e-12


def test_multibranch_equals_lse_weighted_combine(port):
    """O = sum_b e^{lse_b} O_b / sum_b e^{lse_b} over covering branches."""
    n = 96
    q, k, v = (rand((n, 8), s) for s in (11, 12, 13))
    branches = [(16, 1, 0), (32, 2, 1), (48, 4, 2), (96, 8, 3)]
    mb, lse_mb = port.multibranch(q, k, v, branches)
    num = np.zeros((n, 8))
    den = np.zeros(n)
    for w, r, g in branches:
        o = port.dilated_attention(q, k, v, w, r, g)
        lse = port.dilated_lse(q, k, w, r, g)
        wgt = np.where(np.isfinite(lse), np.exp(lse), 0.0)
        num += wgt[:, None] * o
        den += wgt
    cov = den > 0
    assert np.abs(mb[cov] - num[cov] / den[cov, None]).max() <= 1e-12
    assert (mb[~cov] == 0).all()
    assert np.abs(lse_mb[cov] - np.log(den[cov])).max() <= 1e-12


def test_lse_oracle_definition(port):
    n, w, r, g = 40, 10, 2, 1
    q, k = rand((n, 4), 1), rand((n, 4), 2)
    lse = port.dilated_lse(q, k, w, r, g)
    for i in range(n // w):
        rows = list(range(i * w + g, i * w + w, r))
        for a in rows:
            s = np.array([q[a] @ k[b] for b in rows]) / 2.0
            assert abs(lse[a] - np.log(np.exp(s).sum())) <= 1e-12
    sel = np.zeros(n, bool)
    for i in range(n // w):
        sel[i * w + g: i * w + w: r] = True
    assert np.isneginf(lse[~sel]).all()


def test_batched_oracle_drivers_match_per_head_calls(port):
    """The threaded [B, N, h, d] drivers used by the full-batch GPU parity
    tests run exactly the pinned single-head restatement per (image, head)."""
    rng = np.random.default_rng(5)
    B, n, h, d = 2, 96, 3, 8
    q, k, v = (rng.standard_normal((B, n, h, d)) for _ in range(3))
    offs = [0, 1, 1]
    out = port.dilated_batched(q, k, v, 32, 2, offs, threads=3)
    br = [(32, 1, [0, 0, 0]), (48, 2, offs)]
    mb, mbl = port.multibranch_batched(q, k, v, br, threads=2)
    for b in range(B):
        for j in range(h):
            assert np.array_equal(out[b, :, j], port.dilated_attention(q[b, :, j], k[b, :, j], v[b, :, j], 32, 2,
                                                                       offs[j]))
            o1, l1 = port.multibranch(q[b, :, j], k[b, :, j], v[b, :, j], [(w, r, g[j]) for w, r, g in br])
            assert np.array_equal(mb[b, :, j], o1) and np.array_equal(mbl[b, j], l1)
