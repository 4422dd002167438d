"""dfa_gemm -- the layers' GEMM (tcgen05 for bf16, SIMT for f32) with its
epilogue (bias, residual, erf GELU) -- against a plain PyTorch fp32
reference of the same op on the same (bf16-rounded) inputs.  Covers tile
edges (M, N, K not multiples of 128 / BN / 64), every tile width the
dispatcher picks (64, 128, 192, 256), strided-batch operands with the
offset-class split's row strides, and a shared (batch-stride 0) weight.

Tolerance: fp32 accumulation of bf16 products, bf16 output -> max error
<= 1e-2 x max|ref| (bf16 keeps 8 bits; the accumulation order differs);
f32 SIMT path <= 1e-5 x max|ref|."""
import pytest

pytestmark = pytest.mark.gpu


def _torch():
    import torch

    return torch


def _ref(a, b, bias=None, c=None, beta=1.0, gelu=False):
    torch = _torch()
    y = a.float() @ b.float()
    if bias is not None:
        y = y + bias.float()
    if c is not None:
        y = y + beta * c.float()
    if gelu:
        y = 0.5 * y * (1.0 + torch.erf(y / 2 ** 0.5))
    return y


def _close(got, want, dtype):
    torch = _torch()
    tol = 1e-2 if dtype == torch.bfloat16 else 1e-5
    err = (got.float() - want).abs().max().item()
    scale = max(1.0, want.abs().max().item())
    assert err <= tol * scale, (err, scale)


CASES = [
    # M, N, K, bias, residual, gelu
    (128, 64, 64, False, False, False),
    (1000, 576, 384, False, False, False),   # class-split QKV shape (N = 3 x 192), M tail
    (300, 192, 200, True, False, False),     # K tail (200 = 3 x 64 + 8), BN = 192
    (513, 384, 384, True, True, False),      # wo + bo + residual, BN = 192
    (4096, 1536, 384, True, False, True),    # w1 + b1 + GELU, BN = 256
    (4096, 384, 1536, True, True, False),    # w2 + b2 + residual, long K
    (257, 320, 64, False, False, True),      # N = 320 -> BN = 64, GELU
    (64, 1000, 128, True, False, False),     # N tail (1000 = 3 x 256 + 232)
]


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("M,N,K,bias,res,gelu", CASES)
def test_gemm_vs_torch(dfa, cuda, dtype, M, N, K, bias, res, gelu):
    torch = _torch()
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    a = torch.randn((M, K), device="cuda", generator=g).to(dt)
    b = (torch.randn((K, N), device="cuda", generator=g) / K ** 0.5).to(dt)
    bi = torch.randn((N,), device="cuda", generator=g).to(dt) if bias else None
    c = torch.randn((M, N), device="cuda", generator=g).to(dt) if res else None
    out = dfa.gemm(a, b, bias=bi, c=c, gelu=gelu)
    torch.cuda.synchronize()
    _close(out[0], _ref(a, b, bi, c, 1.0, gelu), dt)
    assert dfa.last_launch_count() == 1


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_gemm_class_split_strides(dfa, cuda, dtype):
    """The offset-class split's two GEMMs: (1) A = rows g mod r of x (row
    stride r D, batch = class at element offset g D), B = the class's column
    block of the packed weights (batch stride 3 hd), D per class back to
    back; (2) D written to rows g mod r of out (row stride r D) with bias and
    a residual read through the same strides."""
    torch = _torch()
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    r, Mr, D, hd = 2, 700, 384, 192
    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.randn((Mr * r, D), device="cuda", generator=g).to(dt)
    wp = (torch.randn((D, 3 * D), device="cuda", generator=g) / D ** 0.5).to(dt)
    qkv = torch.empty((r, Mr, 3 * hd), device="cuda", dtype=dt)
    lib = dfa.lib
    dfa._check(lib.dfa_gemm(dfa._dtype_code(x), r, Mr, 3 * hd, D, x.data_ptr(), r * D, D, wp.data_ptr(), 3 * D,
                            3 * hd, qkv.data_ptr(), 3 * hd, Mr * 3 * hd, None, 0, 0.0, None, 0, dfa._stream_ptr(None)))
    for cls in range(r):
        _close(qkv[cls], _ref(x[cls::r], wp[:, cls * 3 * hd:(cls + 1) * 3 * hd]), dt)
    att = torch.randn((r, Mr, hd), device="cuda", generator=g).to(dt)
    wo = (torch.randn((r, hd, D), device="cuda", generator=g) / hd ** 0.5).to(dt)
    bo = torch.randn((D,), device="cuda", generator=g).to(dt)
    resid = torch.randn((Mr * r, D), device="cuda", generator=g).to(dt)
    out = torch.full((Mr * r, D), float("nan"), device="cuda", dtype=dt)
    dfa._check(lib.dfa_gemm(dfa._dtype_code(x), r, Mr, D, hd, att.data_ptr(), hd, Mr * hd, wo.data_ptr(), D, hd * D,
                            out.data_ptr(), r * D, D, resid.data_ptr(), r * D, 1.0, bo.data_ptr(), 0,
                            dfa._stream_ptr(None)))
    torch.cuda.synchronize()
    for cls in range(r):
        _close(out[cls::r], _ref(att[cls], wo[cls], bo, resid[cls::r]), dt)


def test_gemm_shared_weight_batch(dfa, cuda):
    """batch > 1 with B's batch stride 0: every entry multiplies the same weight."""
    torch = _torch()
    g = torch.Generator(device="cuda").manual_seed(3)
    a = torch.randn((3, 200, 128), device="cuda", generator=g).to(torch.bfloat16)
    b = (torch.randn((128, 256), device="cuda", generator=g) / 128 ** 0.5).to(torch.bfloat16)
    out = dfa.gemm(a, b)
    torch.cuda.synchronize()
    for i in range(3):
        _close(out[i], _ref(a[i], b), torch.bfloat16)
