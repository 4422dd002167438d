"""Parity of the CUDA path (through the C-ABI) against the CPU oracle.

Tolerances (BASELINE.json north_star):
  * index permutation of the gather/scatter: bit-exact;
  * fp32 validation mode: max-abs <= 1e-4;
  * bf16 in/out with fp32 accumulate: max-abs <= 2e-2 and
    mean relative error sum|err| / sum|ref| <= 1e-2.
The bf16 tests give the oracle the SAME bf16-rounded inputs upcast to f64.
"""
import numpy as np
import pytest

from conftest import rand

pytestmark = pytest.mark.gpu

F32_TOL = 1e-4
BF16_MAX_ABS = 2e-2
BF16_MEAN_REL = 1e-2


def _torch():
    import torch

    return torch


def to_dev(x, dtype):
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(x)).to(device="cuda", dtype=dtype)


def bf16_round(x):
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


def oracle_batched(port, q, k, v, w, r, offsets):
    """q, k [B, N, h, d], v [B, N, h, dv] float64 -> oracle out [B, N, h, dv]."""
    B, N, h, _ = q.shape
    out = np.zeros(v.shape)
    for b in range(B):
        for j in range(h):
            out[b, :, j] = port.dilated_attention(q[b, :, j], k[b, :, j], v[b, :, j], w, r, offsets[j])
    return out


def run(dfa, q, k, v, cfg, dtype, lse=False):
    torch = _torch()
    td = torch.float32 if dtype == "f32" else torch.bfloat16
    qd, kd, vd = to_dev(q, td), to_dev(k, td), to_dev(v, td)
    L = torch.empty((q.shape[0], q.shape[2], q.shape[1]), dtype=torch.float32, device="cuda") if lse else None
    o = dfa.dfa_forward(qd, kd, vd, cfg, lse=L)
    torch.cuda.synchronize()
    o = o.to(torch.float64).cpu().numpy()
    return (o, L.cpu().numpy()) if lse else o


def errors(got, want):
    err = np.abs(got - want)
    return err.max(), err.sum() / max(np.abs(want).sum(), 1e-30)


def make_cfg(dfa, n, w, r, h, d, offsets=None, dv=0):
    offs = offsets if offsets is not None else dfa.AttentionConfig.spread_offsets(h, r)
    return dfa.AttentionConfig(n, w, r, h, d, list(offs), value_dim=dv)


# -------------------------------------------------------------- fp32 SIMT
SMALL = [
    # (N, w, r, h, d, dv): tails, r !| w, empty views, d != dv, single rows
    (8, 4, 2, 2, 4, 4), (10, 4, 2, 2, 4, 4), (16, 8, 4, 4, 8, 8), (33, 7, 3, 3, 8, 5), (100, 30, 4, 4, 16, 16),
    (12, 12, 1, 1, 4, 4), (1, 1, 1, 1, 8, 8), (64, 16, 2, 2, 32, 32), (257, 64, 4, 4, 64, 64),
    (300, 300, 1, 1, 128, 128), (200, 64, 8, 8, 200, 100), (40, 9, 4, 4, 8, 8),
]


@pytest.mark.parametrize("n,w,r,h,d,dv", SMALL)
def test_simt_f32_small(dfa, port, cuda, n, w, r, h, d, dv):
    B = 2
    q, k = rand((B, n, h, d), n * 7 + 1), rand((B, n, h, d), n * 7 + 2)
    v = rand((B, n, h, dv), n * 7 + 3)
    cfg = make_cfg(dfa, n, w, r, h, d, dv=dv)
    got = run(dfa, q.astype(np.float32), k.astype(np.float32), v.astype(np.float32), cfg, "f32")
    want = oracle_batched(port, q, k, v, w, r, cfg.head_offsets)
    assert errors(got, want)[0] <= F32_TOL


def test_headline_f32_config1(dfa, port, ref, cuda):
    """BASELINE config 1: B=1, h=1, N=4096, w=512, r=2, d=64, gamma=0, fp32."""
    q, k, v = (rand((4096, 64), s, np.float32) for s in (901, 902, 903))
    cfg = dfa.AttentionConfig(4096, 512, 2, 1, 64, [0])
    got = dfa.dilated_attention(to_dev(q, _torch().float32), to_dev(k, _torch().float32),
                                to_dev(v, _torch().float32), cfg, 0).cpu().numpy()
    want32 = ref.dilated_attention(q, k, v, 512, 2, 0)
    want64 = port.dilated_attention(q.astype(np.float64), k.astype(np.float64), v.astype(np.float64), 512, 2, 0)
    assert np.abs(got - want32).max() <= F32_TOL
    assert np.abs(got - want64).max() <= F32_TOL
    # rows no view selects are exact zeros
    assert (got[1::2] == 0).all()


# -------------------------------------------------------- bf16 tcgen05
def _bf16_case(dfa, port, B, n, w, r, h, seed, offsets=None):
    q, k, v = (bf16_round(rand((B, n, h, 64), seed + s)) for s in range(3))
    cfg = make_cfg(dfa, n, w, r, h, 64, offsets)
    assert dfa.query_path(cfg, "bf16", B) == 1, "tcgen05 path not selected"
    got = run(dfa, q, k, v, cfg, "bf16")
    want = oracle_batched(port, q, k, v, w, r, cfg.head_offsets)
    return errors(got, want)


def test_tcgen05_config2_slice(dfa, port, cuda):
    """Config 2 layout [B, N, 6, 64], gamma_j = j mod 2, bf16 (B reduced for oracle time)."""
    mx, rel = _bf16_case(dfa, port, 4, 4096, 512, 2, 6, 100)
    assert mx <= BF16_MAX_ABS and rel <= BF16_MEAN_REL, (mx, rel)


SWEEP = [(w, r) for w in (256, 512, 1024, 2048, 4096) for r in (1, 2, 4, 8)]


@pytest.mark.parametrize("w,r", SWEEP)
def test_tcgen05_branch_sweep(dfa, port, cuda, w, r):
    """Config 4 (w, r) grid at h=6, offsets j mod r (partial coverage for r=8)."""
    mx, rel = _bf16_case(dfa, port, 1, 4096, w, r, 6, 7 * w + r)
    assert mx <= BF16_MAX_ABS and rel <= BF16_MEAN_REL, (w, r, mx, rel)


@pytest.mark.parametrize("n,w,r,h", [
    (1000, 300, 2, 2),   # m = 150 (not a multiple of 128), tail segment m = 50
    (512, 64, 2, 2),     # m = 32: four segments per 128-row tile (block-diagonal)
    (768, 96, 1, 1),     # m = 96
    (640, 640, 1, 1),    # one segment, m = 640 (5 key tiles, online softmax)
    (4104, 513, 3, 3),   # m = 171, tail
    (130, 130, 2, 2),    # T = 65 < 128: partial query tile
    (4096, 4096, 1, 1),  # whole sequence, 32 key tiles
])
def test_tcgen05_geometry_edges(dfa, port, cuda, n, w, r, h):
    mx, rel = _bf16_case(dfa, port, 2, n, w, r, h, n + w)
    assert mx <= BF16_MAX_ABS and rel <= BF16_MEAN_REL, (mx, rel)


def test_tcgen05_vs_simt_full_config2(dfa, cuda):
    """Full config 2 (B=64, h=6): the two independent device kernels agree."""
    torch = _torch()
    from paper_2403_09195_b200 import _lib, path_override

    g = torch.Generator(device="cuda").manual_seed(5)
    q, k, v = (torch.randn((64, 4096, 6, 64), device="cuda", generator=g, dtype=torch.bfloat16) for _ in range(3))
    cfg = make_cfg(dfa, 4096, 512, 2, 6, 64)
    a = dfa.dfa_forward(q, k, v, cfg)
    with path_override(_lib.DFA_PATH_SIMT):
        b = dfa.dfa_forward(q, k, v, cfg)
    torch.cuda.synchronize()
    err = (a.float() - b.float()).abs()
    assert err.max().item() <= BF16_MAX_ABS
    assert (err.sum() / b.float().abs().sum()).item() <= BF16_MEAN_REL


# --------------------------------------------- bit-exact index permutation
def _permutation_inputs(B, n, h, seed):
    """Keys = queries = +/-8 patterns with margin: each query's softmax is an
    exact one-hot on itself, so O must equal V at the same row, bit for bit."""
    rng = np.random.default_rng(seed)
    qk = np.where(rng.random((B, n, h, 64)) < 0.5, -8.0, 8.0)
    # nonzero integers: an exact-zero V row would expose the ~1e-28 weights of
    # the other keys, everything else rounds them away.
    v = (rng.integers(1, 257, size=(B, n, h, 64)) * np.where(rng.random((B, n, h, 64)) < 0.5, -1, 1)).astype(
        np.float64)
    return qk, v


@pytest.mark.parametrize("n,w,r,h,path", [
    (4096, 512, 2, 6, "tcgen05"), (1000, 300, 2, 2, "tcgen05"), (512, 64, 4, 4, "tcgen05"),
    (4096, 512, 2, 6, "simt"), (10, 4, 2, 2, "simt"), (33, 7, 3, 3, "simt"),
])
def test_index_permutation_bit_exact(dfa, cuda, n, w, r, h, path):
    torch = _torch()
    from paper_2403_09195_b200 import _lib, path_override

    B = 2
    qk, v = _permutation_inputs(B, n, h, n + r)
    cfg = make_cfg(dfa, n, w, r, h, 64)
    # margin check: self score beats every other score in the view by > 64 (x 1/8 scale)
    qd, vd = to_dev(qk, torch.bfloat16), to_dev(v, torch.bfloat16)
    mode = _lib.DFA_PATH_SM100_TCGEN05 if path == "tcgen05" else _lib.DFA_PATH_SIMT
    with path_override(mode):
        o = dfa.dfa_forward(qd, qd, vd, cfg)
    torch.cuda.synchronize()
    got = o.to(torch.float64).cpu().numpy()
    want = np.zeros_like(v)
    for j, g in enumerate(cfg.head_offsets):
        for i in range(cfg.num_segments()):
            rows = dfa.make_segment_view(n, w, r, i, g).row_indices
            sub = qk[:, rows, j]
            s = np.einsum("bid,bjd->bij", sub, sub)
            np.einsum("bii->bi", s)[...] = -np.inf
            assert (s.max(axis=2) < 64 * 64 - 512).all(), "permutation inputs lack margin"
            want[:, rows, j] = v[:, rows, j]
    assert np.array_equal(got, want)


# ------------------------------------------------------------- properties
def test_determinism_bitwise(dfa, cuda):
    """Disjoint writes, no atomics: repeated runs are bit-identical (gate 8)."""
    torch = _torch()
    g = torch.Generator(device="cuda").manual_seed(1)
    q, k, v = (torch.randn((8, 4096, 6, 64), device="cuda", generator=g, dtype=torch.bfloat16) for _ in range(3))
    cfg = make_cfg(dfa, 4096, 512, 2, 6, 64)
    a = dfa.dfa_forward(q, k, v, cfg).clone()
    b = dfa.dfa_forward(q, k, v, cfg)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


def test_zero_rows_and_full_coverage(dfa, cuda):
    """Head j writes only rows of class gamma_j; h >= r covers every row."""
    torch = _torch()
    q, k, v = (torch.randn((2, 4096, 6, 64), device="cuda", dtype=torch.bfloat16) for _ in range(3))
    cfg = make_cfg(dfa, 4096, 512, 4, 6, 64)  # offsets 0,1,2,3,0,1
    o = dfa.dfa_forward(q, k, v, cfg).float()
    for j, g in enumerate(cfg.head_offsets):
        rows = torch.arange(4096, device="cuda")
        sel = (rows % 4) == g
        assert (o[:, ~sel, j] == 0).all()
        assert (o[:, sel, j].abs().amax(dim=-1) > 0).all()


def test_lse_output(dfa, port, cuda):
    B, n, w, r, h = 2, 1024, 256, 2, 2
    q, k, v = (bf16_round(rand((B, n, h, 64), 40 + s)) for s in range(3))
    cfg = make_cfg(dfa, n, w, r, h, 64)
    _, L = run(dfa, q, k, v, cfg, "bf16", lse=True)
    for b in range(B):
        for j in range(h):
            want = port.dilated_lse(q[b, :, j], k[b, :, j], w, r, cfg.head_offsets[j])
            fin = np.isfinite(want)
            assert np.array_equal(np.isfinite(L[b, j]), fin)
            assert np.abs(L[b, j][fin] - want[fin]).max() <= 1e-3


def test_fault_hook_is_caught(dfa, port, cuda):
    """attention.hpp:237-241: the parity harness demonstrably fails when armed."""
    q, k, v = (rand((1, 64, 1, 8), s, np.float32) for s in (1, 2, 3))
    cfg = make_cfg(dfa, 64, 16, 2, 1, 8)
    want = oracle_batched(port, q.astype(np.float64), k.astype(np.float64), v.astype(np.float64), 16, 2, [0])
    with dfa.fault_perturb():
        bad = run(dfa, q, k, v, cfg, "f32")
    good = run(dfa, q, k, v, cfg, "f32")
    assert errors(bad, want)[0] > F32_TOL
    assert errors(good, want)[0] <= F32_TOL


def test_host_entry_point_matches_device(dfa, cuda):
    """dfa_forward_host (H2D + kernel + D2H inside the C-ABI) == device call."""
    torch = _torch()
    cfg = make_cfg(dfa, 4096, 512, 2, 6, 64)
    q, k, v = (torch.randn((4, 4096, 6, 64), dtype=torch.bfloat16).pin_memory() for _ in range(3))
    out = torch.empty_like(q).pin_memory()
    ws = dfa.Workspace(dfa.Workspace.bytes_for(cfg, "bf16", 4))
    dfa.dfa_forward_host(q, k, v, out, cfg, ws)
    dev = dfa.dfa_forward(q.cuda(), k.cuda(), v.cuda(), cfg).cpu()
    assert torch.equal(out, dev)


def test_reference_shaped_errors(dfa, cuda):
    torch = _torch()
    cfg = dfa.AttentionConfig(16, 8, 2, 1, 4, [0])
    x = torch.zeros((16, 4), device="cuda")
    with pytest.raises(dfa.OutOfRange):
        dfa.dilated_attention(x, x, x, cfg, 2)
    with pytest.raises(dfa.DimensionError):
        dfa.dilated_attention(x, torch.zeros((16, 5), device="cuda"), x, cfg, 0)
    with pytest.raises(dfa.DimensionError):
        dfa.dilated_attention(x, x, torch.zeros((15, 4), device="cuda"), cfg, 0)
    with pytest.raises(dfa.DimensionError):
        dfa.dilated_attention(torch.zeros((15, 4), device="cuda"), x, x, cfg, 0)
    with pytest.raises(dfa.ConfigError):
        dfa.dilated_attention(x, x, x, dfa.AttentionConfig(16, 17, 1, 1, 4, [0]), 0)
    with pytest.raises(dfa.DimensionError):
        dfa.dilated_attention(x.cpu(), x.cpu(), x.cpu(), cfg, 0)


def test_single_query_passes_value_through(dfa, cuda):
    """test_attention.cpp:56-63 / :212-221: m = 1 => output row == v row."""
    torch = _torch()
    cfg = dfa.AttentionConfig(4, 4, 4, 1, 4, [1])
    q, k, v = (torch.randn((4, 4), device="cuda") for _ in range(3))
    o = dfa.dilated_attention(q, k, v, cfg, 1)
    assert torch.equal(o[1], v[1])
    assert (o[[0, 2, 3]] == 0).all()


# ------------------------------------------- multi-(w, r) LSE combine (ext.)
def test_multibranch_single_branch_is_dfa_forward(dfa, cuda):
    """One branch: weights e^0 = 1, so the combine returns dfa_forward bit for bit."""
    torch = _torch()
    for dt in (torch.bfloat16, torch.float32):
        q, k, v = (torch.randn((2, 1024, 2, 64), device="cuda", dtype=dt) for _ in range(3))
        cfg = make_cfg(dfa, 1024, 256, 2, 2, 64)
        a = dfa.dfa_forward(q, k, v, cfg)
        b = dfa.dfa_forward_multibranch(q, k, v, cfg, [(256, 2)])
        torch.cuda.synchronize()
        assert torch.equal(a, b), dt


@pytest.mark.parametrize("branches", [
    [(512, 1), (1024, 2), (2048, 4), (4096, 8)],  # LongNet-style geometric set
    [(256, 2), (512, 2), (1024, 4)],
])
def test_multibranch_vs_oracle(dfa, port, cuda, branches):
    """LSE-weighted combine vs the extension oracle (one dense softmax over the
    multiset of keys the covering branches select); bf16 tolerances."""
    torch = _torch()
    B, n, h = 1, 4096, 2
    q, k, v = (bf16_round(rand((B, n, h, 64), 70 + s)) for s in range(3))
    cfg = make_cfg(dfa, n, branches[0][0], branches[0][1], h, 64)
    qd, kd, vd = (to_dev(x, torch.bfloat16) for x in (q, k, v))
    L = torch.empty((B, h, n), dtype=torch.float32, device="cuda")
    o = dfa.dfa_forward_multibranch(qd, kd, vd, cfg, branches, lse=L)
    torch.cuda.synchronize()
    got = o.double().cpu().numpy()
    Lg = L.cpu().numpy()
    want = np.zeros_like(got)
    for j in range(h):
        brs = [(w, r, j % r) for w, r in branches]
        ob, lb = port.multibranch(q[0, :, j], k[0, :, j], v[0, :, j], brs)
        want[0, :, j] = ob
        fin = np.isfinite(lb)
        assert np.array_equal(np.isfinite(Lg[0, j]), fin)
        assert np.abs(Lg[0, j][fin] - lb[fin]).max() <= 2e-3
    mx, rel = errors(got, want)
    assert mx <= BF16_MAX_ABS and rel <= BF16_MEAN_REL, (mx, rel)


@pytest.mark.timeout(120)
@pytest.mark.parametrize("w,r", [(256, 2), (256, 4), (256, 8), (512, 4), (512, 8), (1024, 8), (512, 2), (4096, 1)])
def test_tcgen05_many_units_per_cta(dfa, cuda, w, r):
    """B=64, h=6: ~20 work units per persistent CTA (the protocol's steady
    state, incl. one-step-per-slot units when m <= 128) vs the SIMT kernel."""
    torch = _torch()
    from paper_2403_09195_b200 import _lib, path_override

    g = torch.Generator(device="cuda").manual_seed(w + r)
    q, k, v = (torch.randn((64, 4096, 6, 64), device="cuda", generator=g, dtype=torch.bfloat16) for _ in range(3))
    cfg = make_cfg(dfa, 4096, w, r, 6, 64)
    a = dfa.dfa_forward(q, k, v, cfg)
    with path_override(_lib.DFA_PATH_SIMT):
        b = dfa.dfa_forward(q, k, v, cfg)
    torch.cuda.synchronize()
    err = (a.float() - b.float()).abs()
    assert err.max().item() <= BF16_MAX_ABS
    assert (err.sum() / b.float().abs().sum()).item() <= BF16_MEAN_REL


@pytest.mark.parametrize("branches", [
    [(512, 1), (1024, 2), (2048, 4), (4096, 8)],
    [(4096, 8), (256, 4), (512, 1)],  # sparse first branch: later merges land on zero rows
    [(256, 2), (256, 2)],             # duplicate branch: weights 1/2 each, o unchanged
])
def test_multibranch_fused_epilogue_matches_unfused(dfa, cuda, branches):
    """bf16 per-branch path (branch 0 writes o + running lse, later branches merge
    in their epilogue: one launch per branch, no combine kernel) vs the unfused
    path (per-branch o_b/lse_b + combine kernel, forced via the SIMT override)."""
    torch = _torch()
    from paper_2403_09195_b200 import _lib, multibranch_mode, path_override

    g = torch.Generator(device="cuda").manual_seed(len(branches))
    B, n, h = 4, 4096, 6
    q, k, v = (torch.randn((B, n, h, 64), device="cuda", generator=g, dtype=torch.bfloat16) for _ in range(3))
    cfg = make_cfg(dfa, n, 512, 1, h, 64)
    L1 = torch.empty((B, h, n), dtype=torch.float32, device="cuda")
    with multibranch_mode(_lib.DFA_MB_PER_BRANCH):
        a = dfa.dfa_forward_multibranch(q, k, v, cfg, branches, lse=L1)
        assert dfa.last_launch_count() == len(branches)
    L2 = torch.empty_like(L1)
    with path_override(_lib.DFA_PATH_SIMT):
        b = dfa.dfa_forward_multibranch(q, k, v, cfg, branches, lse=L2)
    torch.cuda.synchronize()
    err = (a.float() - b.float()).abs()
    assert err.max().item() <= BF16_MAX_ABS
    assert (err.sum() / b.float().abs().sum()).item() <= BF16_MEAN_REL
    fin = torch.isfinite(L2)
    assert torch.equal(torch.isfinite(L1), fin)
    assert (L1[fin] - L2[fin]).abs().max().item() <= 2e-3
    # rows no branch selects are exactly zero
    assert (a.float()[~fin.permute(0, 2, 1)] == 0).all()
    if branches[0] == branches[1]:
        c = dfa.dfa_forward(q, k, v, make_cfg(dfa, n, 256, 2, h, 64))
        assert (a.float() - c.float()).abs().max().item() <= 1e-2


def test_multibranch_fault_hook_once(dfa, cuda):
    """The recompose fault hook perturbs the combined output once."""
    torch = _torch()
    q, k, v = (torch.randn((1, 1024, 2, 64), device="cuda", dtype=torch.bfloat16) for _ in range(3))
    cfg = make_cfg(dfa, 1024, 256, 2, 2, 64)
    br = [(256, 2), (512, 4)]
    a = dfa.dfa_forward_multibranch(q, k, v, cfg, br)
    with dfa.fault_perturb():
        b = dfa.dfa_forward_multibranch(q, k, v, cfg, br)
    torch.cuda.synchronize()
    d = (b.float() - a.float()).flatten()
    assert d[1:].abs().max().item() == 0.0
    assert abs(d[0].item() - 1e-3) <= 8e-3  # bf16 rounding of o[0] + 1e-3


@pytest.mark.parametrize("dt,w,r", [("bf16", 512, 2), ("bf16", 256, 4), ("f32", 512, 2), ("bf16", 300, 3)])
def test_strided_qkv_equals_contiguous(dfa, cuda, dt, w, r):
    """dfa_forward_strided on q|k|v column blocks of one [B, N, 3, h, d]
    buffer (the fused projection output) is bit-identical to dfa_forward on
    contiguous copies, on both device paths."""
    torch = _torch()
    td = torch.float32 if dt == "f32" else torch.bfloat16
    B, n, h, d = 2, 1200 if w == 300 else 2048, 6, 64
    g = torch.Generator(device="cuda").manual_seed(w * r)
    qkv = torch.randn((B, n, 3, h, d), device="cuda", dtype=td, generator=g)
    cfg = make_cfg(dfa, n, w, r, h, d)
    L1 = torch.empty((B, h, n), dtype=torch.float32, device="cuda")
    L2 = torch.empty_like(L1)
    a = dfa.dfa_forward_strided(qkv, cfg, lse=L1)
    q, k, v = (qkv[:, :, i].contiguous() for i in range(3))
    b = dfa.dfa_forward(q, k, v, cfg, lse=L2)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    assert torch.equal(L1, L2)


def test_host_entry_zero_copy_equals_copy_path(dfa, cuda):
    """dfa_forward_host with pinned inputs reads the kept rows straight from
    host memory (zero-copy TMA); with a pinned o it also writes only the kept
    output rows in place (host threads zero-fill the rest).  Every mode --
    kept-out, device output + D2H, copy-in, pageable -- gives the same bits on
    a NaN-poisoned o, and the reported PCIe bytes shrink to the kept rows."""
    torch = _torch()
    B, n, h = 8, 4096, 6
    cfg = make_cfg(dfa, n, 512, 2, h, 64)
    g = torch.Generator().manual_seed(3)
    q, k, v = (torch.randn((B, n, h, 64), generator=g).to(torch.bfloat16) for _ in range(3))
    pq, pk, pv = (t.pin_memory() for t in (q, k, v))
    ws = dfa.Workspace(dfa.Workspace.bytes_for(cfg, "bf16", B))
    full = 3 * q.numel() * 2
    outs = []
    # (inputs, zero-copy in, pinned o, kept-out mode) -> expected (h2d, d2h)
    modes = [((pq, pk, pv), True, True, True, (full // 2, q.numel())),
             ((pq, pk, pv), True, True, False, (full // 2, 2 * q.numel())),
             ((pq, pk, pv), True, False, True, (full // 2, 2 * q.numel())),
             ((pq, pk, pv), False, True, True, (full, 2 * q.numel())),
             ((q, k, v), True, True, True, (full, 2 * q.numel()))]
    for args, zc, pinned_o, kept, want in modes:
        o = torch.full_like(q, float("nan"))
        if pinned_o:
            o = o.pin_memory()
        with dfa.host_zero_copy(zc), dfa.host_kept_out(kept):
            dfa.dfa_forward_host(*args, o, cfg, ws)
            assert dfa.host_transfer_bytes(*args, cfg, out=o) == want
        outs.append(o)
    ws.close()
    ref = dfa.dfa_forward(q.cuda(), k.cuda(), v.cuda(), cfg).cpu()
    for o in outs:
        assert torch.equal(o, ref)


@pytest.mark.parametrize("n,w,r,offs,with_lse", [
    (4096, 1024, 4, [3, 1, 2, 0, 1, 3], True),   # r = 4, custom offsets, lse through the host call
    (2048, 2048, 8, [0, 7, 7, 2, 5, 1], False),  # one segment, r = 8: 7 / 8 of o zero-filled on the host
    (2304, 512, 2, [0, 1, 0, 1, 0, 1], True),    # tail segment
])
def test_host_kept_out_zero_fill(dfa, cuda, n, w, r, offs, with_lse):
    """Kept-out mode: the host zero fill covers exactly the rows no view keeps
    (NaN-poisoned pinned o), lse comes back alongside."""
    torch = _torch()
    B, h = 3, 6
    cfg = dfa.AttentionConfig(n, w, r, h, 64, offs)
    g = torch.Generator().manual_seed(n + r)
    q, k, v = (torch.randn((B, n, h, 64), generator=g).to(torch.bfloat16).pin_memory() for _ in range(3))
    o = torch.full((B, n, h, 64), float("nan")).to(torch.bfloat16).pin_memory()
    L = torch.full((B, h, n), float("nan")).pin_memory() if with_lse else None
    ws = dfa.Workspace(dfa.Workspace.bytes_for(cfg, "bf16", B, with_lse=with_lse))
    dfa.dfa_forward_host(q, k, v, o, cfg, ws, lse=L)
    ws.close()
    Lr = torch.empty((B, h, n), device="cuda") if with_lse else None
    ref = dfa.dfa_forward(q.cuda(), k.cuda(), v.cuda(), cfg, lse=Lr).cpu()
    assert torch.equal(o, ref)
    if with_lse:
        assert torch.equal(L, Lr.cpu())


def test_forward_and_backward_from_a_fresh_thread(dfa, cuda):
    """The tcgen05 launchers encode TMA descriptors with the driver API; a
    thread whose first CUDA call that is (e.g. PyTorch's autograd worker)
    must still get the device's context (ensure_context)."""
    import threading

    torch = _torch()
    cfg = make_cfg(dfa, 1024, 256, 2, 2, 64)
    g = torch.Generator(device="cuda").manual_seed(3)
    q, k, v, do = (torch.randn((1, 1024, 2, 64), generator=g, device="cuda", dtype=torch.bfloat16) for _ in range(4))
    L = torch.empty((1, 2, 1024), dtype=torch.float32, device="cuda")
    ref = dfa.dfa_forward(q, k, v, cfg, lse=L)
    ref_g = dfa.dfa_backward(q, k, v, ref, L, do, cfg)
    torch.cuda.synchronize()
    out = {}

    def work():
        try:
            out["o"] = dfa.dfa_forward(q, k, v, cfg)
            out["g"] = dfa.dfa_backward(q, k, v, ref, L, do, cfg)
            torch.cuda.synchronize()
        except Exception as e:  # surfaced below
            out["err"] = e

    t = threading.Thread(target=work)
    t.start()
    t.join()
    assert "err" not in out, out.get("err")
    assert torch.equal(out["o"], ref)
    for a, b in zip(out["g"], ref_g):
        assert torch.equal(a, b)


def test_host_kept_out_repeatable(dfa, cuda):
    """Kept-out host mode run 10 times on the same pinned buffers (the host
    zero fill runs concurrently with the kernel's in-place writes): identical
    bits every time, equal to the device path."""
    torch = _torch()
    B, n, h = 16, 4096, 6
    cfg = make_cfg(dfa, n, 512, 2, h, 64)
    g = torch.Generator().manual_seed(19)
    q, k, v = (torch.randn((B, n, h, 64), generator=g).to(torch.bfloat16).pin_memory() for _ in range(3))
    o = torch.empty_like(q).pin_memory()
    ws = dfa.Workspace(dfa.Workspace.bytes_for(cfg, "bf16", B))
    ref = dfa.dfa_forward(q.cuda(), k.cuda(), v.cuda(), cfg).cpu()
    for _ in range(10):
        o.fill_(float("nan"))
        dfa.dfa_forward_host(q, k, v, o, cfg, ws)
        assert torch.equal(o, ref)
    ws.close()
