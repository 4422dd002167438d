"""Backward of the dilated core.

CPU: the C restatement (oracle_dilated_backward_f64) is bit-identical to the
reference's own autodiff tape run on the dilated branch of attention_mix
(ref_dilated_backward_f64 -> ag::backward), on edge geometries.
GPU (-m gpu): dfa_backward through the C-ABI vs that oracle -- fp32 within
1e-4 (relative to the gradient scale), bf16 within the bf16 tolerances --
plus the autograd wrapper and determinism."""
import numpy as np
import pytest

from conftest import rand

GEOMS = [  # n, w, r, gamma, d, dv
    (64, 16, 2, 1, 8, 8), (100, 30, 4, 3, 16, 16), (64, 64, 1, 0, 8, 8), (50, 50, 3, 2, 5, 7),
    (40, 12, 5, 4, 8, 8),  # tail segment, empty views (gamma >= tail rows)
    (256, 64, 2, 0, 64, 64),
]


@pytest.mark.parametrize("n,w,r,g,d,dv", GEOMS)
def test_port_backward_equals_reference_tape(port, ref, n, w, r, g, d, dv):
    q, k, do = rand((n, d), 1), rand((n, d), 2), rand((n, dv), 4)
    v = rand((n, dv), 3)
    a = port.dilated_backward(q, k, v, do, w, r, g)
    b = ref.dilated_backward(q, k, v, do, w, r, g)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_port_backward_matches_finite_differences(port):
    """Independent check of the restated math: central differences of
    sum(O * dO) (acceptance.cpp:206-339 checks the tape the same way)."""
    n, w, r, g, d = 24, 8, 2, 1, 4
    q, k, v, do = (rand((n, d), s) for s in range(4))
    gq, gk, gv = port.dilated_backward(q, k, v, do, w, r, g)
    loss = lambda q_, k_, v_: float((port.dilated_attention(q_, k_, v_, w, r, g) * do).sum())  # noqa: E731
    eps = 1e-6
    for which, grad in ((0, gq), (1, gk), (2, gv)):
        for idx in [(1, 0), (3, 2), (5, 3), (0, 1)]:
            args = [q.copy(), k.copy(), v.copy()]
            args[which][idx] += eps
            up = loss(*args)
            args[which][idx] -= 2 * eps
            dn = loss(*args)
            assert abs((up - dn) / (2 * eps) - grad[idx]) <= 1e-7 * max(1.0, abs(grad[idx]))


# ------------------------------------------------------------------- GPU
def _oracle_batched_bwd(port, q, k, v, do, w, r, offsets):
    B, N, h, d = q.shape
    gq, gk, gv = np.zeros(q.shape), np.zeros(k.shape), np.zeros(v.shape)
    for b in range(B):
        for j in range(h):
            a = port.dilated_backward(q[b, :, j], k[b, :, j], v[b, :, j], do[b, :, j], w, r, offsets[j])
            gq[b, :, j], gk[b, :, j], gv[b, :, j] = a
    return gq, gk, gv


BWD_CASES = [  # B, n, h, w, r, d, dv
    (2, 256, 2, 64, 2, 64, 64), (1, 100, 3, 30, 4, 16, 16), (1, 40, 1, 12, 5, 8, 8), (1, 1024, 2, 256, 2, 64, 64),
    (1, 96, 2, 48, 3, 32, 48), (1, 512, 1, 512, 1, 128, 128),
]


@pytest.mark.gpu
@pytest.mark.parametrize("B,n,h,w,r,d,dv", BWD_CASES)
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_backward_vs_oracle(dfa, port, cuda, B, n, h, w, r, d, dv, dtype):
    import torch

    td = torch.float32 if dtype == "f32" else torch.bfloat16
    offs = [j % r for j in range(h)]
    cfg = dfa.AttentionConfig(n, w, r, h, d, offs, value_dim=dv)
    q, k, v, do = rand((B, n, h, d), 11), rand((B, n, h, d), 12), rand((B, n, h, dv), 13), rand((B, n, h, dv), 14)
    dev = [torch.from_numpy(x).to("cuda", td) for x in (q, k, v, do)]
    if dtype == "bf16":  # the oracle sees the same rounded inputs
        q, k, v, do = (t.double().cpu().numpy() for t in dev)
    L = torch.empty((B, h, n), dtype=torch.float32, device="cuda")
    o = dfa.dfa_forward(dev[0], dev[1], dev[2], cfg, lse=L)
    gq, gk, gv = dfa.dfa_backward(dev[0], dev[1], dev[2], o, L, dev[3], cfg)
    assert dfa.last_launch_count() in (2, 3)  # tcgen05 (delta + 1) or SIMT (delta + 2)
    torch.cuda.synchronize()
    want = _oracle_batched_bwd(port, q, k, v, do, w, r, offs)
    for got, ref_ in zip((gq, gk, gv), want):
        got = got.double().cpu().numpy()
        err = np.abs(got - ref_)
        scale = max(1.0, np.abs(ref_).max())
        if dtype == "f32":
            assert err.max() <= 1e-4 * scale, err.max()
        else:
            assert err.max() <= 2e-2 * scale, err.max()
            assert err.sum() / max(np.abs(ref_).sum(), 1e-30) <= 1e-2
    # rows no view selects: exact zero gradients
    sel = np.zeros((n, h), dtype=bool)
    for j, gmm in enumerate(offs):
        for s0 in range(0, n, w):
            sel[s0 + gmm:min(s0 + w, n):r, j] = True
    for t in (gq, gk, gv):
        assert (t.float().cpu().numpy()[:, ~sel] == 0).all()


@pytest.mark.gpu
def test_backward_deterministic_and_autograd(dfa, cuda):
    import torch

    B, n, h, w, r, d = 2, 1024, 6, 512, 2, 64
    cfg = dfa.AttentionConfig(n, w, r, h, d, [j % r for j in range(h)])
    g = torch.Generator(device="cuda").manual_seed(5)
    q, k, v = (torch.randn((B, n, h, d), device="cuda", generator=g, dtype=torch.bfloat16).requires_grad_()
               for _ in range(3))
    o = dfa.dilated_attention_fn(q, k, v, cfg)
    go = torch.randn_like(o)
    o.backward(go)
    grads = [t.grad.clone() for t in (q, k, v)]
    for t in (q, k, v):
        t.grad = None
    dfa.dilated_attention_fn(q, k, v, cfg).backward(go)
    for a, t in zip(grads, (q, k, v)):
        assert torch.equal(a, t.grad)  # bitwise deterministic (no atomics)
    # vs torch autograd of a plain fp64 restatement (test-only reference)
    qd, kd, vd = (t.detach().double().requires_grad_() for t in (q, k, v))
    out = torch.zeros((B, n, h, d), dtype=torch.float64, device="cuda")
    for j in range(h):
        gm = j % r
        for s0 in range(0, n, w):
            idx = torch.arange(s0 + gm, min(s0 + w, n), r, device="cuda")
            s = torch.einsum("bid,bjd->bij", qd[:, idx, j], kd[:, idx, j]) / d ** 0.5
            out[:, idx, j] = torch.einsum("bij,bjd->bid", torch.softmax(s, -1), vd[:, idx, j])
    out.backward(go.double())
    for a, t in zip(grads, (qd, kd, vd)):
        err = (a.double() - t.grad).abs()
        assert err.max().item() <= 2e-2 * max(1.0, t.grad.abs().max().item())
        assert (err.sum() / t.grad.abs().sum()).item() <= 1e-2


@pytest.mark.gpu
@pytest.mark.timeout(120)
@pytest.mark.parametrize("w,r,B", [(512, 2, 4), (256, 1, 2), (256, 2, 4), (1024, 4, 2), (512, 4, 2), (2048, 8, 1),
                                   (512, 1, 1), (1024, 2, 1), (4096, 8, 1), (2048, 2, 1),
                                   (256, 4, 2), (256, 8, 2), (512, 8, 2), (128, 8, 1)])
def test_tcgen05_backward_vs_simt(dfa, cuda, w, r, B):
    """bf16 tcgen05 backward -- fused kernel for m = w/r in {128, 256} and for
    m in {16, 32, 64} packed 128 / m segments per tile with a block-diagonal
    mask, the dkdv_long + dq_long pair for m >= 512 -- vs the SIMT backward on the same
    inputs (path override), h = 6, offsets j mod r; and determinism."""
    import torch
    from paper_2403_09195_b200 import _lib, path_override

    n, h, d = 4096, 6, 64
    cfg = dfa.AttentionConfig(n, w, r, h, d, [j % r for j in range(h)])
    g = torch.Generator(device="cuda").manual_seed(w + r)
    q, k, v, do = (torch.randn((B, n, h, d), device="cuda", generator=g, dtype=torch.bfloat16) for _ in range(4))
    L = torch.empty((B, h, n), dtype=torch.float32, device="cuda")
    o = dfa.dfa_forward(q, k, v, cfg, lse=L)
    a = dfa.dfa_backward(q, k, v, o, L, do, cfg)
    assert dfa.last_launch_count() == (2 if w // r <= 256 else 3)  # delta + fused, or delta + dkdv + dq
    a2 = dfa.dfa_backward(q, k, v, o, L, do, cfg)
    with path_override(_lib.DFA_PATH_SIMT):
        b = dfa.dfa_backward(q, k, v, o, L, do, cfg)
        assert dfa.last_launch_count() == 3
    torch.cuda.synchronize()
    for x, x2, y in zip(a, a2, b):
        assert torch.equal(x, x2)
        err = (x.float() - y.float()).abs()
        scale = max(1.0, y.float().abs().max().item())
        assert err.max().item() <= 2e-2 * scale, err.max().item()
        assert (err.sum() / y.float().abs().sum()).item() <= 1e-2


@pytest.mark.gpu
@pytest.mark.timeout(300)
@pytest.mark.parametrize("w,r,B", [(512, 2, 64), (256, 1, 16), (256, 2, 16), (64, 1, 16)])
def test_tcgen05_backward_repeatable_under_load(dfa, cuda, w, r, B):
    """Stress: 30 back-to-back backward launches at bench scale give bitwise
    identical gradients.  Two-block views exercise the dV read-before-overwrite
    ordering at key-block transitions, one-block views the double-buffered
    operand slots, (64, 1) the packed-segment instantiation."""
    import torch

    n, h = 4096, 6
    cfg = dfa.AttentionConfig(n, w, r, h, 64, [j % r for j in range(h)])
    g = torch.Generator(device="cuda").manual_seed(w + r)
    q, k, v, do = (torch.randn((B, n, h, 64), device="cuda", generator=g, dtype=torch.bfloat16) for _ in range(4))
    L = torch.empty((B, h, n), device="cuda")
    o = dfa.dfa_forward(q, k, v, cfg, lse=L)
    ws = torch.empty(B * h * n * 4 + 256, dtype=torch.uint8, device="cuda")
    ref = [torch.empty_like(q) for _ in range(3)]
    dfa.dfa_backward(q, k, v, o, L, do, cfg, *ref, workspace=ws)
    got = [torch.empty_like(q) for _ in range(3)]
    for _ in range(30):
        dfa.dfa_backward(q, k, v, o, L, do, cfg, *got, workspace=ws)
    torch.cuda.synchronize()
    for a, b in zip(ref, got):
        assert torch.equal(a, b)
