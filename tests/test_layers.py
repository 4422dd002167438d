"""Callers either side of the core, on the GPU through
the C-ABI, against the compiled reference:
  * dfa_multi_head_dilated vs attnkit::multi_head_dilated (attention.hpp:340-360);
  * dfa_encoder_block_forward vs one block of encoder_forward run on the
    reference's own ops (encoder.hpp:241-248 via ref_encoder_block_f64).
fp32 (validation mode, SIMT core + SIMT fp32 GEMM, no TF32): <= 1e-4
relative to the output scale.  bf16: <= 2e-2 max-abs relative to the output
scale and <= 1e-2 mean relative error, oracle fed the same bf16-rounded
inputs and weights."""
import numpy as np
import pytest

from conftest import rand

pytestmark = pytest.mark.gpu


def _dev(x, dtype):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dtype)


def _round(x, dtype):
    import torch

    return _dev(x, dtype).double().cpu().numpy()


def _check(got, want, dtype):
    err = np.abs(got - want)
    scale = max(1.0, np.abs(want).max())
    if dtype == "f32":
        assert err.max() <= 1e-4 * scale, err.max()
    else:
        assert err.max() <= 2e-2 * scale, err.max()
        assert err.sum() / np.abs(want).sum() <= 1e-2, err.sum() / np.abs(want).sum()


@pytest.mark.parametrize("n,h,d,w,r,B", [(256, 2, 64, 64, 2, 2), (1024, 6, 64, 256, 2, 1), (100, 4, 16, 30, 3, 1)])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_multi_head_vs_reference(dfa, ref, cuda, n, h, d, w, r, B, dtype):
    import torch

    td = torch.float32 if dtype == "f32" else torch.bfloat16
    D = h * d
    x = rand((B, n, D), 31)
    ws = [rand((h, D, d), 32 + i) / np.sqrt(D) for i in range(3)]
    wo = rand((D, D), 35) / np.sqrt(D)
    if dtype == "bf16":
        x, wo = _round(x, td), _round(wo, td)
        ws = [_round(a, td) for a in ws]
    cfg = dfa.AttentionConfig(n, w, r, h, d, dfa.AttentionConfig.spread_offsets(h, r))
    out = dfa.multi_head_dilated(_dev(x, td), *[_dev(a, td) for a in ws], _dev(wo, td), cfg)
    torch.cuda.synchronize()
    got = out.double().cpu().numpy()
    for b in range(B):
        want = ref.multi_head_dilated(x[b], ws[0], ws[1], ws[2], wo, w, r)
        _check(got[b], want, dtype)


def test_multi_head_requires_full_coverage(dfa, cuda):
    import torch

    cfg = dfa.AttentionConfig(64, 16, 4, 2, 8, [0, 1])  # classes 2, 3 uncovered
    x = torch.zeros((1, 64, 16), device="cuda")
    w = torch.zeros((2, 16, 8), device="cuda")
    with pytest.raises(dfa.ConfigError, match="covered by no head"):
        dfa.multi_head_dilated(x, w, w, w, torch.zeros((16, 16), device="cuda"), cfg)


def _block_weights(D, h, hidden, seed):
    d = D // h
    s = 1.0 / np.sqrt(D)
    rng = np.random.default_rng(seed)
    return {
        "ln1_g": 1 + 0.1 * rng.standard_normal(D), "ln1_b": 0.1 * rng.standard_normal(D),
        "wq": s * rng.standard_normal((h, D, d)), "wk": s * rng.standard_normal((h, D, d)),
        "wv": s * rng.standard_normal((h, D, d)), "wo": s * rng.standard_normal((D, D)),
        "bo": 0.1 * rng.standard_normal(D), "ln2_g": 1 + 0.1 * rng.standard_normal(D),
        "ln2_b": 0.1 * rng.standard_normal(D), "w1": s * rng.standard_normal((D, hidden)),
        "b1": 0.1 * rng.standard_normal(hidden), "w2": rng.standard_normal((hidden, D)) / np.sqrt(hidden),
        "b2": 0.1 * rng.standard_normal(D),
    }


@pytest.mark.parametrize("n,h,d,w,r,B", [(256, 2, 64, 64, 2, 2), (1024, 6, 64, 256, 2, 1), (64, 4, 16, 16, 2, 1),
                                        (256, 12, 64, 64, 2, 1), (256, 4, 64, 64, 4, 2)])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_encoder_block_vs_reference(dfa, ref, cuda, n, h, d, w, r, B, dtype):
    import torch

    td = torch.float32 if dtype == "f32" else torch.bfloat16
    D, hidden = h * d, 4 * h * d
    p = _block_weights(D, h, hidden, 41)
    x = rand((B, n, D), 40)
    if dtype == "bf16":
        x = _round(x, td)
        p = {k: _round(v, td) for k, v in p.items()}
    cfg = dfa.AttentionConfig(n, w, r, h, d, dfa.AttentionConfig.spread_offsets(h, r))
    out = dfa.encoder_block_forward(_dev(x, td), {k: _dev(v, td) for k, v in p.items()}, cfg)
    assert dfa.last_launch_count() >= 7  # LN, QKV, core, wo, LN, w1 + GELU (epilogue), w2
    torch.cuda.synchronize()
    got = out.double().cpu().numpy()
    for b in range(B):
        want = ref.encoder_block(x[b], p, h, w, r)
        _check(got[b], want, dtype)


@pytest.mark.parametrize("n,h,w,r,offsets", [
    (512, 4, 128, 2, [1, 0, 0, 1]),          # classes not in head order
    (512, 3, 128, 2, [0, 0, 1]),             # uneven classes (2 + 1 heads)
    (1024, 8, 512, 4, [3, 2, 1, 0, 0, 1, 2, 3]),
    (768, 6, 256, 2, [0, 1, 0, 1, 0, 1]),
])
def test_multi_head_offset_classes_bf16(dfa, ref, cuda, n, h, w, r, offsets):
    """The bf16 layer runs per offset class (heads grouped by gamma_j, 1/r of
    the projection work, csrc/dfa_api.cpp class_split_layer): any assignment
    of heads to classes with full coverage matches the reference."""
    import torch

    d, B = 64, 2
    D = h * d
    x = rand((B, n, D), 61)
    ws = [rand((h, D, d), 62 + i) / np.sqrt(D) for i in range(3)]
    wo = rand((D, D), 65) / np.sqrt(D)
    td = torch.bfloat16
    x, wo = _round(x, td), _round(wo, td)
    ws = [_round(a, td) for a in ws]
    cfg = dfa.AttentionConfig(n, w, r, h, d, offsets)
    out = dfa.multi_head_dilated(_dev(x, td), *[_dev(a, td) for a in ws], _dev(wo, td), cfg)
    torch.cuda.synchronize()
    got = out.double().cpu().numpy()
    for b in range(B):
        want = ref.multi_head_dilated(x[b], ws[0], ws[1], ws[2], wo, w, r, offsets)
        _check(got[b], want, "bf16")
