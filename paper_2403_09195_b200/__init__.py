"""B200-native Dilated Flash Attention (SAM-Lightening, arxiv 2403.09195).

Host-side mirror of the reference operator API for the hot path
(/root/reference/proj/include/attnkit/attention.hpp), calling the sm_100a
kernels through the C-ABI in include/dfa.h (libdfa.so):

    AttentionConfig            attention.hpp:24-66
    make_segment_view          attention.hpp:84-98
    dilated_attention          attention.hpp:280-301  (single head, [N, d])
    dfa_forward                batched multi-head [B, N, h, d] (the device API)
    flop_count / flop_csv_*    attention.hpp:370-394
    fault_perturb              attention.hpp:237-241

Errors mirror the reference's exception taxonomy (common.hpp:13-30):
ConfigError, DimensionError, ContractError and OutOfRange (an IndexError,
the std::out_of_range analogue).  PyTorch is used only for device memory and
streams; every forward runs a CUDA kernel from libdfa.so -- there is no CPU
path, and a CPU tensor is rejected.
"""
from __future__ import annotations

import contextlib
import ctypes
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

from . import _lib
from ._lib import lib

__all__ = [
    "AttentionConfig",
    "SegmentView",
    "FlopCount",
    "ConfigError",
    "DimensionError",
    "ContractError",
    "OutOfRange",
    "CudaError",
    "UnsupportedError",
    "make_segment_view",
    "flop_count",
    "flop_csv_header",
    "flop_csv_row",
    "dilated_attention",
    "dfa_forward",
    "dfa_forward_host",
    "dfa_forward_multibranch",
    "query_path",
    "fault_perturb",
    "last_launch_count",
]


class DfaError(RuntimeError):
    """Base of the errors raised by the C-ABI."""


class ConfigError(DfaError):
    """attnkit::config_error."""


class DimensionError(DfaError):
    """attnkit::dimension_error."""


class ContractError(DfaError):
    """attnkit::contract_error."""


class OutOfRange(IndexError):
    """std::out_of_range (segment index / offset outside its range)."""


class CudaError(DfaError):
    """A CUDA runtime/driver failure inside the library."""


class UnsupportedError(DfaError):
    """A valid configuration the device kernels do not implement."""


class TensorIOError(DfaError):
    """attnkit::io_error (DTNSR1 tensor files)."""


_ERRORS = {
    _lib.DFA_ERR_CONFIG: ConfigError,
    _lib.DFA_ERR_DIMENSION: DimensionError,
    _lib.DFA_ERR_OUT_OF_RANGE: OutOfRange,
    _lib.DFA_ERR_CONTRACT: ContractError,
    _lib.DFA_ERR_CUDA: CudaError,
    _lib.DFA_ERR_UNSUPPORTED: UnsupportedError,
    _lib.DFA_ERR_IO: TensorIOError,
}


def _check(status: int) -> None:
    if status != _lib.DFA_OK:
        msg = lib.dfa_last_error().decode()
        raise _ERRORS.get(status, DfaError)(msg)


@dataclass
class AttentionConfig:
    """attention.hpp:24-33.  kernel is "naive" or "tiled" (validated; the GPU always tiles)."""

    seq_len: int = 0
    segment_len: int = 0
    interval: int = 1
    num_heads: int = 1
    head_dim: int = 0
    head_offsets: List[int] = field(default_factory=list)
    kernel: str = "naive"
    tile_size: int = 1
    scale_scores: bool = True
    value_dim: int = 0  # 0 => d_v = d (the reference infers d_v from v)

    def num_segments(self) -> int:
        return (self.seq_len + self.segment_len - 1) // self.segment_len

    def model_dim(self) -> int:
        return self.num_heads * self.head_dim

    @staticmethod
    def spread_offsets(heads: int, interval: int) -> List[int]:
        """attention.hpp:38-42: gamma_j = j mod r."""
        return [j % interval for j in range(heads)]

    def _c(self):
        n = max(1, len(self.head_offsets), self.num_heads)
        offs = (ctypes.c_int64 * n)(*[int(g) for g in self.head_offsets])
        kern = {"naive": 0, "tiled": 1}.get(self.kernel, -1)
        c = _lib.DfaConfig(
            self.seq_len,
            self.segment_len,
            self.interval,
            self.num_heads,
            self.head_dim,
            self.value_dim,
            ctypes.cast(offs, ctypes.POINTER(ctypes.c_int64)) if self.head_offsets else None,
            kern,
            self.tile_size,
            1 if self.scale_scores else 0,
        )
        c._keep = offs  # keep the offsets array alive with the struct
        return c

    def validate(self, require_full_coverage: bool = False) -> None:
        """attention.hpp:44-65; raises ConfigError with the reference's message."""
        if len(self.head_offsets) != self.num_heads:
            raise ConfigError(f"attention: {len(self.head_offsets)} offsets for {self.num_heads} heads")
        c = self._c()
        _check(lib.dfa_validate(ctypes.byref(c), 1 if require_full_coverage else 0))


@dataclass
class SegmentView:
    """attention.hpp:70-76."""

    segment_index: int
    offset: int
    row_indices: List[int]


def make_segment_view(seq_len: int, segment_len: int, interval: int, segment_index: int, offset: int) -> SegmentView:
    """attention.hpp:84-98 (via the C-ABI)."""
    count = ctypes.c_int64(0)
    _check(lib.dfa_segment_view(seq_len, segment_len, interval, segment_index, offset, None, 0, ctypes.byref(count)))
    rows = (ctypes.c_int64 * max(1, count.value))()
    _check(lib.dfa_segment_view(seq_len, segment_len, interval, segment_index, offset, rows, count.value,
                                ctypes.byref(count)))
    return SegmentView(segment_index, offset, list(rows[: count.value]))


@dataclass
class FlopCount:
    """attention.hpp:364-368 (multiplications only)."""

    dense_mults: int
    dilated_mults: int
    ratio: float


def flop_count(cfg: AttentionConfig) -> FlopCount:
    """attention.hpp:370-387."""
    if len(cfg.head_offsets) != cfg.num_heads:
        cfg.validate()
    c = cfg._c()
    dn, dl, rt = ctypes.c_uint64(0), ctypes.c_uint64(0), ctypes.c_double(0)
    _check(lib.dfa_flop_count(ctypes.byref(c), ctypes.byref(dn), ctypes.byref(dl), ctypes.byref(rt)))
    return FlopCount(dn.value, dl.value, rt.value)


def flop_csv_header() -> str:
    """attention.hpp:389."""
    return "N,w,r,h,d,dense_mults,dilated_mults,ratio"


def _fmt_double(x: float) -> str:
    # std::ostream default formatting (%g with 6 significant digits).
    return f"{x:g}"


def flop_csv_row(cfg: AttentionConfig, fc: FlopCount) -> str:
    """attention.hpp:391-394."""
    return (f"{cfg.seq_len},{cfg.segment_len},{cfg.interval},{cfg.num_heads},{cfg.head_dim},"
            f"{fc.dense_mults},{fc.dilated_mults},{_fmt_double(fc.ratio)}")


# ----------------------------------------------------------------- device API
def _torch():
    import torch  # noqa: WPS433 -- torch is plumbing (device memory, streams)

    return torch


def _dtype_code(t) -> int:
    torch = _torch()
    if t.dtype == torch.float32:
        return _lib.DFA_F32
    if t.dtype == torch.bfloat16:
        return _lib.DFA_BF16
    if t.dtype == torch.float64:
        return _lib.DFA_F64
    raise DimensionError(f"dfa: unsupported dtype {t.dtype} (float32, bfloat16 or float64)")


def _code(dtype: str) -> int:
    """"f32" | "bf16" | "f64" -> DFA_* code."""
    try:
        return {"f32": _lib.DFA_F32, "bf16": _lib.DFA_BF16, "f64": _lib.DFA_F64}[dtype]
    except KeyError:
        raise ConfigError(f"dfa: unknown dtype {dtype!r} (f32, bf16 or f64)") from None


def _stream_ptr(stream) -> int:
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


def query_path(cfg: AttentionConfig, dtype: str = "bf16", batch: int = 1) -> int:
    """Which device kernel dfa_forward takes (DFA_PATH_* in include/dfa.h)."""
    c = cfg._c()
    out = ctypes.c_int32(0)
    _check(lib.dfa_query_path(ctypes.byref(c), _code(dtype), batch,
                              ctypes.byref(out)))
    return out.value


def last_launch_count() -> int:
    return int(lib.dfa_last_launch_count())


def _check_qkv(q, k, v, cfg: AttentionConfig, who: str):
    """Shape / dtype / device checks shared by every device entry point (the
    C-ABI trusts cfg for sizes, so a mismatch here would read or write out of
    bounds instead of raising).  Returns (B, N, h, d, d_v)."""
    for name, t in (("q", q), ("k", k), ("v", v)):
        if not t.is_cuda:
            raise DimensionError(f"{who}: {name} is not a CUDA tensor (no CPU path)")
        if t.dim() != 4:
            raise DimensionError(f"{who}: {name} must be [B, N, h, d], got {tuple(t.shape)}")
        if not t.is_contiguous():
            raise DimensionError(f"{who}: {name} must be contiguous")
        if t.device != q.device:
            raise DimensionError(f"{who}: q, k, v are on different devices")
    B, N, h, d = q.shape
    dv = v.shape[3]
    if tuple(k.shape) != (B, N, h, d):
        raise DimensionError(f"{who}: query/key shape mismatch {tuple(q.shape)} vs {tuple(k.shape)}")
    if tuple(v.shape[:3]) != (B, N, h):
        raise DimensionError(f"{who}: key/value shape mismatch {tuple(k.shape)} vs {tuple(v.shape)}")
    if q.dtype != k.dtype or q.dtype != v.dtype:
        raise DimensionError(f"{who}: q, k, v dtypes differ")
    if N != cfg.seq_len:
        raise DimensionError(f"{who}: expected {cfg.seq_len} rows, got {N}")
    if h != cfg.num_heads or len(cfg.head_offsets) != h:
        raise ConfigError(f"attention: {len(cfg.head_offsets)} offsets for {h} heads")
    if d != cfg.head_dim:
        raise DimensionError(f"{who}: head_dim {cfg.head_dim} but q has width {d}")
    return B, N, h, d, dv


def _check_buffer(t, shape, dtype, device, who: str, name: str):
    """A caller-supplied output / gradient buffer: exact shape, dtype, device, contiguous."""
    if (tuple(t.shape) != tuple(shape) or t.dtype != dtype or not t.is_cuda or t.device != device
            or not t.is_contiguous()):
        raise DimensionError(f"{who}: {name} must be a contiguous {dtype} CUDA tensor of shape {tuple(shape)} "
                             f"on {device}, got {tuple(t.shape)} {t.dtype} on {t.device}")


def dfa_forward(q, k, v, cfg: AttentionConfig, out=None, lse=None, stream=None):
    """Batched multi-head forward: q, k [B, N, h, d], v [B, N, h, d_v] (CUDA,
    contiguous, float32 or bfloat16) -> o [B, N, h, d_v].  Head j uses offset
    cfg.head_offsets[j].  `lse`: optional float32 [B, h, N] output tensor."""
    torch = _torch()
    B, N, h, d, dv = _check_qkv(q, k, v, cfg, "dfa_forward")
    if out is None:
        out = torch.empty((B, N, h, dv), dtype=q.dtype, device=q.device)
    else:
        _check_buffer(out, (B, N, h, dv), q.dtype, q.device, "dfa_forward", "out")
    if lse is not None:
        _check_buffer(lse, (B, h, N), torch.float32, q.device, "dfa_forward", "lse")
    c = cfg._c()
    c.value_dim = dv
    _check(lib.dfa_forward(ctypes.byref(c), _dtype_code(q), B, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                           out.data_ptr(), lse.data_ptr() if lse is not None else None, _stream_ptr(stream)))
    return out


def dfa_forward_strided(qkv, cfg: AttentionConfig, out=None, lse=None, stream=None):
    """Core on a fused projection output qkv [B, N, 3, h, d] (q | k | v column
    blocks per token, token stride 3 h d) -> o [B, N, h, d] (dfa_forward_strided)."""
    torch = _torch()
    if not qkv.is_cuda or not qkv.is_contiguous() or qkv.dim() != 5 or qkv.shape[2] != 3:
        raise DimensionError("dfa_forward_strided: qkv must be a contiguous CUDA [B, N, 3, h, d] tensor")
    B, N, _, h, d = qkv.shape
    if N != cfg.seq_len:
        raise DimensionError(f"dfa_forward_strided: expected {cfg.seq_len} rows, got {N}")
    if h != cfg.num_heads or len(cfg.head_offsets) != h:
        raise ConfigError(f"attention: {len(cfg.head_offsets)} offsets for {h} heads")
    if d != cfg.head_dim:
        raise DimensionError(f"dfa_forward_strided: head_dim {cfg.head_dim} but qkv has width {d}")
    if out is None:
        out = torch.empty((B, N, h, d), dtype=qkv.dtype, device=qkv.device)
    else:
        _check_buffer(out, (B, N, h, d), qkv.dtype, qkv.device, "dfa_forward_strided", "out")
    if lse is not None:
        _check_buffer(lse, (B, h, N), torch.float32, qkv.device, "dfa_forward_strided", "lse")
    c = cfg._c()
    es = qkv.element_size()
    base = qkv.data_ptr()
    ld = 3 * h * d
    _check(lib.dfa_forward_strided(ctypes.byref(c), _dtype_code(qkv), B, base, ld, base + h * d * es, ld,
                                   base + 2 * h * d * es, ld, out.data_ptr(), out.stride(1),
                                   lse.data_ptr() if lse is not None else None, _stream_ptr(stream)))
    return out


def dilated_attention(q, k, v, cfg: AttentionConfig, head_offset: int, workers: int = 1, stream=None):
    """attention.hpp:280-301 on CUDA tensors: q, k [N, d], v [N, d_v] -> [N, d_v].

    Same checks and error types as the reference: cfg.validate(); q/k widths
    and k/v rows must agree (require_qkv :102-110); q and k need cfg.seq_len
    rows (:285-286); head_offset in [0, r) else OutOfRange (:287-288).
    `workers` is accepted and ignored (the GPU grid replaces parallel_for)."""
    del workers
    cfg.validate()
    for name, t in (("q", q), ("k", k), ("v", v)):
        if t.dim() != 2:
            raise DimensionError(f"dilated_attention: expected rank-2 tensor, got {list(t.shape)}")
    if q.shape[1] != k.shape[1]:
        raise DimensionError(f"dilated_attention: query/key width mismatch {list(q.shape)} vs {list(k.shape)}")
    if k.shape[0] != v.shape[0]:
        raise DimensionError(f"dilated_attention: key/value row mismatch {list(k.shape)} vs {list(v.shape)}")
    if q.shape[0] != cfg.seq_len or k.shape[0] != cfg.seq_len:
        raise DimensionError(f"dilated_attention: expected {cfg.seq_len} rows, got {q.shape[0]}")
    if head_offset < 0 or head_offset >= cfg.interval:
        raise OutOfRange(f"dilated_attention: head offset {head_offset} outside [0, {cfg.interval})")
    one = AttentionConfig(cfg.seq_len, cfg.segment_len, cfg.interval, 1, q.shape[1], [head_offset], cfg.kernel,
                          cfg.tile_size, cfg.scale_scores)
    N, d = q.shape
    out = dfa_forward(q.contiguous().view(1, N, 1, d), k.contiguous().view(1, N, 1, d),
                      v.contiguous().view(1, N, 1, v.shape[1]), one, stream=stream)
    return out.view(N, v.shape[1])


class Workspace:
    """Device staging buffer for the host-buffer entry points (dfa_workspace_t)."""

    def __init__(self, nbytes: int):
        self.handle = ctypes.c_void_p(0)
        self.nbytes = nbytes
        _check(lib.dfa_workspace_create(nbytes, ctypes.byref(self.handle)))

    @staticmethod
    def bytes_for(cfg: AttentionConfig, dtype: str, batch: int, with_lse: bool = False) -> int:
        c = cfg._c()
        out = ctypes.c_size_t(0)
        _check(lib.dfa_workspace_bytes(ctypes.byref(c), _code(dtype), batch,
                                       1 if with_lse else 0, ctypes.byref(out)))
        return out.value

    def close(self) -> None:
        if self.handle:
            lib.dfa_workspace_destroy(self.handle)
            self.handle = ctypes.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 -- interpreter teardown
            pass


def dfa_forward_host(q, k, v, out, cfg: AttentionConfig, ws: Workspace, dtype: str = "bf16", lse=None, stream=None):
    """End-to-end call on HOST tensors (pinned CPU torch tensors or anything
    exposing data_ptr()): H2D, forward, D2H, synchronize -- all inside the
    C-ABI (dfa_forward_host)."""
    B = q.shape[0]
    c = cfg._c()
    c.value_dim = v.shape[-1]
    code = _code(dtype)
    sp = _stream_ptr(stream) if stream is not None else None
    _check(lib.dfa_forward_host(ctypes.byref(c), code, B, q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                                lse.data_ptr() if lse is not None else None, ws.handle, sp))
    return out


@contextlib.contextmanager
def host_zero_copy(enabled: bool):
    """Scope dfa_forward_host's zero-copy input mode (default on)."""
    lib.dfa_set_host_zero_copy(1 if enabled else 0)
    try:
        yield
    finally:
        lib.dfa_set_host_zero_copy(1)


@contextlib.contextmanager
def host_kept_out(enabled: bool):
    """Scope dfa_forward_host's kept-rows-out mode for a pinned host o (default on)."""
    lib.dfa_set_host_kept_out(1 if enabled else 0)
    try:
        yield
    finally:
        lib.dfa_set_host_kept_out(1)


def host_transfer_bytes(q, k, v, cfg: AttentionConfig, dtype: str = "bf16", with_lse: bool = False, out=None):
    """(h2d, d2h) bytes dfa_forward_host moves for these host tensors (out: the
    host output buffer -- kept rows only cross PCIe when it is pinned)."""
    c = cfg._c()
    c.value_dim = v.shape[-1]
    h2d, d2h = ctypes.c_size_t(0), ctypes.c_size_t(0)
    _check(lib.dfa_host_transfer_bytes(ctypes.byref(c), _code(dtype),
                                       q.shape[0], q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                       out.data_ptr() if out is not None else None, 1 if with_lse else 0,
                                       ctypes.byref(h2d), ctypes.byref(d2h)))
    return h2d.value, d2h.value


def dfa_forward_multibranch(q, k, v, cfg: AttentionConfig, branches, out=None, lse=None, stream=None,
                            workspace=None):
    """EXTENSION: LSE-weighted combine of several (w, r) branches (include/dfa.h).
    `branches`: list of (w, r) or (w, r, head_offsets); offsets default to
    j mod r.  cfg supplies N, h, d, scale_scores.  Returns o [B, N, h, d_v]."""
    torch = _torch()
    B, N, h, d, dv = _check_qkv(q, k, v, cfg, "dfa_forward_multibranch")
    bs, keep = [], []
    for br in branches:
        w, r = br[0], br[1]
        offs = list(br[2]) if len(br) > 2 else AttentionConfig.spread_offsets(h, r)
        if len(offs) != h:
            raise ConfigError(f"attention: {len(offs)} offsets for {h} heads (branch w={w}, r={r})")
        arr = (ctypes.c_int64 * h)(*offs)
        keep.append(arr)
        bs.append(_lib.DfaBranch(w, r, ctypes.cast(arr, ctypes.POINTER(ctypes.c_int64))))
    barr = (_lib.DfaBranch * len(bs))(*bs)
    c = cfg._c()
    c.value_dim = dv
    code = _dtype_code(q)
    need = ctypes.c_size_t(0)
    _check(lib.dfa_multibranch_workspace_bytes(ctypes.byref(c), len(bs), code, B, ctypes.byref(need)))
    if workspace is None or workspace.numel() < need.value:
        workspace = torch.empty(need.value, dtype=torch.uint8, device=q.device)
    if out is None:
        out = torch.empty((B, N, h, dv), dtype=q.dtype, device=q.device)
    else:
        _check_buffer(out, (B, N, h, dv), q.dtype, q.device, "dfa_forward_multibranch", "out")
    if lse is not None:
        _check_buffer(lse, (B, h, N), torch.float32, q.device, "dfa_forward_multibranch", "lse")
    _check(lib.dfa_forward_multibranch(ctypes.byref(c), len(bs), barr, code, B, q.data_ptr(), k.data_ptr(),
                                       v.data_ptr(), out.data_ptr(), lse.data_ptr() if lse is not None else None,
                                       workspace.data_ptr(), workspace.numel(), _stream_ptr(stream)))
    return out


@contextlib.contextmanager
def fault_perturb():
    """attention.hpp:237-241: arm the recompose fault hook inside the block."""
    lib.dfa_set_fault_perturb(1)
    try:
        yield
    finally:
        lib.dfa_set_fault_perturb(0)


@contextlib.contextmanager
def multibranch_mode(mode: int):
    """Test hook: DFA_MB_PER_BRANCH forces one launch per branch (epilogue
    LSE merge) instead of the single fused multi-branch kernel."""
    lib.dfa_set_multibranch_mode(mode)
    try:
        yield
    finally:
        lib.dfa_set_multibranch_mode(0)


@contextlib.contextmanager
def path_override(path: int):
    """Test hook: force DFA_PATH_SIMT or require DFA_PATH_SM100_TCGEN05."""
    lib.dfa_set_path_override(path)
    try:
        yield
    finally:
        lib.dfa_set_path_override(0)


# ------------------------------------------------------------ backward (§8(f) 3)
def dfa_backward(q, k, v, o, lse, do, cfg: AttentionConfig, dq=None, dk=None, dv=None, stream=None,
                 workspace=None):
    """Gradients (dq, dk, dv) of a loss w.r.t. q, k, v given do = dloss/do,
    for o, lse = dfa_forward(q, k, v, cfg, lse=...) (include/dfa.h dfa_backward;
    the reference's tape for the dilated branch of attention_mix,
    encoder.hpp:204-219)."""
    torch = _torch()
    B, N, h, d, dvd = _check_qkv(q, k, v, cfg, "dfa_backward")
    _check_buffer(o, (B, N, h, dvd), q.dtype, q.device, "dfa_backward", "o")
    _check_buffer(do, (B, N, h, dvd), q.dtype, q.device, "dfa_backward", "do")
    _check_buffer(lse, (B, h, N), torch.float32, q.device, "dfa_backward", "lse")
    dq = torch.empty_like(q) if dq is None else dq
    dk = torch.empty_like(k) if dk is None else dk
    dv = torch.empty_like(v) if dv is None else dv
    _check_buffer(dq, tuple(q.shape), q.dtype, q.device, "dfa_backward", "dq")
    _check_buffer(dk, tuple(k.shape), q.dtype, q.device, "dfa_backward", "dk")
    _check_buffer(dv, tuple(v.shape), q.dtype, q.device, "dfa_backward", "dv")
    c = cfg._c()
    c.value_dim = dvd
    need = ctypes.c_size_t(0)
    _check(lib.dfa_backward_workspace_bytes(ctypes.byref(c), B, ctypes.byref(need)))
    if workspace is None or workspace.numel() < need.value:
        workspace = torch.empty(max(need.value, 1), dtype=torch.uint8, device=q.device)
    _check(lib.dfa_backward(ctypes.byref(c), _dtype_code(q), B, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                            o.data_ptr(), lse.data_ptr(), do.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(),
                            workspace.data_ptr(), workspace.numel(), _stream_ptr(stream)))
    return dq, dk, dv


_AUTOGRAD_FN = None


def dilated_attention_fn(q, k, v, cfg: AttentionConfig):
    """Differentiable dfa_forward (torch.autograd.Function over dfa_forward /
    dfa_backward): o = DFA(q, k, v); o.backward(g) fills q/k/v .grad."""
    global _AUTOGRAD_FN
    torch = _torch()
    if _AUTOGRAD_FN is None:
        class _DFA(torch.autograd.Function):
            @staticmethod
            def forward(ctx, q_, k_, v_, cfg_):
                B, N, h, _ = q_.shape
                lse = torch.empty((B, h, N), dtype=torch.float32, device=q_.device)
                o = dfa_forward(q_, k_, v_, cfg_, lse=lse)
                ctx.save_for_backward(q_, k_, v_, o, lse)
                ctx.cfg = cfg_
                return o

            @staticmethod
            def backward(ctx, g):
                q_, k_, v_, o, lse = ctx.saved_tensors
                gq, gk, gv = dfa_backward(q_, k_, v_, o, lse, g.contiguous(), ctx.cfg)
                return gq, gk, gv, None

        _AUTOGRAD_FN = _DFA
    return _AUTOGRAD_FN.apply(q, k, v, cfg)


# ------------------------------------------------- projections / block (§8(f) 1-2)
def _layer_check(x, cfg, who):
    if not x.is_cuda or not x.is_contiguous() or x.dim() != 3:
        raise DimensionError(f"{who}: x must be a contiguous CUDA [B, N, D] tensor")
    D = cfg.num_heads * cfg.head_dim
    if x.shape[1] != cfg.seq_len or x.shape[2] != D:
        raise DimensionError(f"{who}: input {list(x.shape[1:])}, expected [{cfg.seq_len}x{D}]")


def _ws(nbytes, like, workspace):
    torch = _torch()
    if workspace is None or workspace.numel() < nbytes:
        workspace = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=like.device)
    return workspace


def multi_head_dilated(x, wq, wk, wv, wo, cfg: AttentionConfig, out=None, stream=None, workspace=None):
    """attention.hpp:340-360 for a batch: x [B, N, D]; wq/wk/wv [h, D, d]; wo [D, D]."""
    torch = _torch()
    _layer_check(x, cfg, "multi_head_dilated")
    for w_ in (wq, wk, wv, wo):
        if not w_.is_cuda or not w_.is_contiguous() or w_.dtype != x.dtype:
            raise DimensionError("multi_head_dilated: weights must be contiguous CUDA tensors of x's dtype")
    h, D, d = cfg.num_heads, cfg.num_heads * cfg.head_dim, cfg.head_dim
    if tuple(wq.shape) != (h, D, d) or tuple(wk.shape) != (h, D, d) or tuple(wv.shape) != (h, D, d):
        raise DimensionError(f"multi_head_dilated: head projections must be [{h}, {D}, {d}]")
    if tuple(wo.shape) != (D, D):
        raise DimensionError(f"multi_head_dilated: output projection is {list(wo.shape)}, expected [{D}x{D}]")
    B = x.shape[0]
    c = cfg._c()
    need = ctypes.c_size_t(0)
    _check(lib.dfa_multi_head_workspace_bytes(ctypes.byref(c), _dtype_code(x), B, ctypes.byref(need)))
    workspace = _ws(need.value, x, workspace)
    out = torch.empty_like(x) if out is None else out
    _check(lib.dfa_multi_head_dilated(ctypes.byref(c), _dtype_code(x), B, x.data_ptr(), wq.data_ptr(), wk.data_ptr(),
                                      wv.data_ptr(), wo.data_ptr(), out.data_ptr(), workspace.data_ptr(),
                                      workspace.numel(), _stream_ptr(stream)))
    return out


def gemm(a, b, bias=None, c=None, beta=1.0, gelu=False, out=None, stream=None):
    """dfa_gemm: out = epi(a @ b + bias + beta c) for row-major CUDA tensors
    a [.., M, K] (row stride may exceed K), b [.., K, N], c / out [.., M, N];
    a leading batch dim is passed as the batch stride (tensor.hpp:175-195 matmul
    plus the layers' epilogue; bf16 -> tcgen05, float32 -> SIMT)."""
    torch = _torch()
    if a.dim() == 2:
        a, b = a.unsqueeze(0), b.unsqueeze(0) if b.dim() == 2 else b
    batch, M, K = a.shape
    N = b.shape[-1]
    if b.dim() == 2:
        b = b.unsqueeze(0)
    for name, t in (("a", a), ("b", b)):
        if not t.is_cuda or t.stride(-1) != 1:
            raise DimensionError(f"gemm: {name} must be a CUDA tensor with unit column stride")
    if out is None:
        out = torch.empty((batch, M, N), dtype=a.dtype, device=a.device)
    sb = b.stride(0) if b.shape[0] > 1 else 0
    _check(lib.dfa_gemm(_dtype_code(a), batch, M, N, K, a.data_ptr(), a.stride(1), a.stride(0), b.data_ptr(),
                        b.stride(1), sb, out.data_ptr(), out.stride(-2), out.stride(0) if out.dim() == 3 else M * N,
                        c.data_ptr() if c is not None else None, c.stride(-2) if c is not None else 0, beta,
                        bias.data_ptr() if bias is not None else None, 1 if gelu else 0, _stream_ptr(stream)))
    return out


BLOCK_KEYS = ("ln1_g", "ln1_b", "wq", "wk", "wv", "wo", "bo", "ln2_g", "ln2_b", "w1", "b1", "w2", "b2")


def encoder_block_forward(x, weights: dict, cfg: AttentionConfig, out=None, stream=None, workspace=None):
    """One pre-norm encoder block (encoder.hpp:241-248).  weights: BLOCK_KEYS ->
    CUDA tensors of x's dtype (wq/wk/wv [h, D, d], w1 [D, hidden], w2 [hidden, D])."""
    torch = _torch()
    _layer_check(x, cfg, "encoder_block")
    for k_ in BLOCK_KEYS:
        t = weights[k_]
        if not t.is_cuda or not t.is_contiguous() or t.dtype != x.dtype:
            raise DimensionError(f"encoder_block: {k_} must be a contiguous CUDA tensor of x's dtype")
    hidden = weights["w1"].shape[1]
    wt = _lib.DfaBlockWeights(*[weights[k_].data_ptr() for k_ in BLOCK_KEYS], hidden)
    B = x.shape[0]
    c = cfg._c()
    need = ctypes.c_size_t(0)
    _check(lib.dfa_encoder_block_workspace_bytes(ctypes.byref(c), _dtype_code(x), B, hidden, ctypes.byref(need)))
    workspace = _ws(need.value, x, workspace)
    out = torch.empty_like(x) if out is None else out
    _check(lib.dfa_encoder_block_forward(ctypes.byref(c), _dtype_code(x), B, x.data_ptr(), ctypes.byref(wt),
                                         out.data_ptr(), workspace.data_ptr(), workspace.numel(),
                                         _stream_ptr(stream)))
    return out


# ------------------------------------------------------------ DTNSR1 files
def tensor_header(path: str):
    """tensor_io.hpp:97-118: (dtype "f32"|"f64", shape tuple)."""
    dt, rk = ctypes.c_int32(0), ctypes.c_int32(0)
    dims = (ctypes.c_int64 * 8)()
    _check(lib.dfa_tensor_header(os.fsencode(path), ctypes.byref(dt), ctypes.byref(rk), dims))
    return ("f32" if dt.value == 0 else "f64"), tuple(dims[i] for i in range(rk.value))


def load_tensor(path: str, dtype: str = "f64"):
    """load_tensor<Scalar> (tensor_io.hpp:147-153) into a numpy array of `dtype`
    ("f32" | "f64"), converting the stored scalar type like the reference."""
    import numpy as np

    _, shape = tensor_header(path)
    out = np.empty(shape, dtype=np.float32 if dtype == "f32" else np.float64)
    _check(lib.dfa_tensor_load(os.fsencode(path), 0 if dtype == "f32" else 1, out.ctypes.data, out.size))
    return out


def save_tensor(path: str, array) -> None:
    """save_tensor (tensor_io.hpp:86-91); float32 arrays are written as f32,
    everything else as f64 (the format's two dtypes)."""
    import numpy as np

    a = np.asarray(array)
    a = np.asarray(a, dtype=np.float32 if a.dtype == np.float32 else np.float64, order="C")
    dims = (ctypes.c_int64 * max(a.ndim, 1))(*a.shape)
    _check(lib.dfa_tensor_save(os.fsencode(path), 0 if a.dtype == np.float32 else 1, a.ndim, dims,
                               a.ctypes.data if a.size else None))
