"""oracle/oracle.py -- TEST INFRASTRUCTURE ONLY.

numpy/ctypes front end to the two CPU checkers built by oracle/Makefile:

  * ``Port``      -- oracle/liboracle.so, the plain-C restatement of the
                     reference path (dfa_oracle.c; every function cites the
                     reference file:line it restates).
  * ``Reference`` -- oracle/_ref/libattnkit_ref.so, the UNMODIFIED reference
                     headers (/root/reference/proj/include/attnkit) behind
                     extern "C" forwarders (ref_shim.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module -- as the checker or the timed
CPU baseline, never as part of the product path.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libattnkit_ref.so")

_d = ctypes.POINTER(ctypes.c_double)
_f = ctypes.POINTER(ctypes.c_float)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32


def build_port() -> None:
    """(Re)build liboracle.so (gcc; works on the GPU box too)."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def _threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return os.cpu_count() or 1


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"status {code}: {msg}")
        self.code = code


class Port:
    """The C restatement (oracle/dfa_oracle.c)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build_port()
        self.lib = ctypes.CDLL(path)
        L = self.lib
        L.oracle_validate.restype = _i32
        L.oracle_validate.argtypes = [_i64, _i64, _i64, _i64, _i64, _i64p, _i64, _i32, _i64, _i32]
        L.oracle_segment_view.restype = _i32
        L.oracle_segment_view.argtypes = [_i64, _i64, _i64, _i64, _i64, _i64p, _i64, _i64p]
        L.oracle_flop_count.restype = _i32
        L.oracle_flop_count.argtypes = [_i64, _i64, _i64, _i64, _i64, _i64p, ctypes.POINTER(ctypes.c_uint64),
                                        ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_double)]
        for sfx, tp in (("f32", _f), ("f64", _d)):
            fn = getattr(L, f"oracle_dilated_attention_{sfx}")
            fn.restype = _i32
            fn.argtypes = [tp, tp, tp, _i64, _i64, _i64, _i64, _i64, _i64, _i32, _i32, _i64, tp]
        L.oracle_masked_dense_f64.restype = _i32
        L.oracle_masked_dense_f64.argtypes = [_d, _d, _d, _i64, _i64, _i64, _i64, _i64, _i64, _i32, _d]
        L.oracle_dilated_lse_f64.restype = _i32
        L.oracle_dilated_lse_f64.argtypes = [_d, _d, _i64, _i64, _i64, _i64, _i64, _i32, _d]
        L.oracle_multibranch_f64.restype = _i32
        L.oracle_multibranch_f64.argtypes = [_d, _d, _d, _i64, _i64, _i64, _i64, _i64p, _i64p, _i64p, _i32, _d, _d]
        L.oracle_time_dilated_f32.restype = ctypes.c_double
        L.oracle_time_dilated_f32.argtypes = [_f, _f, _f, _i64, _i64, _i64, _i64, _i64, _i64, _f]
        L.oracle_dilated_backward_f64.restype = _i32
        L.oracle_dilated_backward_f64.argtypes = [_d, _d, _d, _d, _i64, _i64, _i64, _i64, _i64, _i64, _i32, _d, _d, _d]
        L.oracle_dilated_batched_f64.restype = _i32
        L.oracle_dilated_batched_f64.argtypes = [_d, _d, _d, _i64, _i64, _i64, _i64, _i64, _i64, _i64, _i64p, _i32, _d]
        L.oracle_multibranch_batched_f64.restype = _i32
        L.oracle_multibranch_batched_f64.argtypes = [_d, _d, _d, _i64, _i64, _i64, _i64, _i64, _i64, _i64p, _i64p,
                                                     _i64p, _i32, _d, _d]

    def validate(self, n, w, r, h, d, offsets, tiled=False, tile=1, full=False) -> int:
        offs = np.asarray(offsets, dtype=np.int64)
        return self.lib.oracle_validate(n, w, r, h, d, _ptr(offs, _i64p), len(offs), int(tiled), tile, int(full))

    def segment_view(self, n, w, r, i, g):
        cnt = ctypes.c_int64(0)
        buf = np.zeros(max(1, (w + r - 1) // r), dtype=np.int64)
        st = self.lib.oracle_segment_view(n, w, r, i, g, _ptr(buf, _i64p), len(buf), ctypes.byref(cnt))
        if st:
            raise OracleError(st)
        return [int(x) for x in buf[: cnt.value]]

    def flop_count(self, n, w, r, h, d, offsets):
        offs = np.asarray(offsets, dtype=np.int64)
        a, b, c = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_double()
        st = self.lib.oracle_flop_count(n, w, r, h, d, _ptr(offs, _i64p), ctypes.byref(a), ctypes.byref(b),
                                        ctypes.byref(c))
        if st:
            raise OracleError(st)
        return a.value, b.value, c.value

    def dilated_attention(self, q, k, v, w, r, gamma, scale=True, tiled=False, tile=1):
        """q, k [N, d], v [N, dv] float32 or float64 -> out [N, dv] (same dtype)."""
        dt = q.dtype
        tp, fn = (_f, self.lib.oracle_dilated_attention_f32) if dt == np.float32 else (
            _d, self.lib.oracle_dilated_attention_f64)
        q, k, v = (np.ascontiguousarray(x, dtype=dt) for x in (q, k, v))
        n, d = q.shape
        dv = v.shape[1]
        out = np.zeros((n, dv), dtype=dt)
        st = fn(_ptr(q, tp), _ptr(k, tp), _ptr(v, tp), n, d, dv, w, r, gamma, int(scale), int(tiled), tile,
                _ptr(out, tp))
        if st:
            raise OracleError(st)
        return out

    def masked_dense(self, q, k, v, w, r, gamma, scale=True):
        q, k, v = (np.ascontiguousarray(x, dtype=np.float64) for x in (q, k, v))
        n, d = q.shape
        out = np.zeros((n, v.shape[1]))
        st = self.lib.oracle_masked_dense_f64(_ptr(q, _d), _ptr(k, _d), _ptr(v, _d), n, d, v.shape[1], w, r, gamma,
                                              int(scale), _ptr(out, _d))
        if st:
            raise OracleError(st)
        return out

    def dilated_lse(self, q, k, w, r, gamma, scale=True):
        q, k = (np.ascontiguousarray(x, dtype=np.float64) for x in (q, k))
        n, d = q.shape
        out = np.zeros(n)
        st = self.lib.oracle_dilated_lse_f64(_ptr(q, _d), _ptr(k, _d), n, d, w, r, gamma, int(scale), _ptr(out, _d))
        if st:
            raise OracleError(st)
        return out

    def multibranch(self, q, k, v, branches, scale=True):
        """branches: list of (w, r, gamma).  Returns (out [N, dv], lse [N])."""
        q, k, v = (np.ascontiguousarray(x, dtype=np.float64) for x in (q, k, v))
        n, d = q.shape
        ws = np.array([b[0] for b in branches], dtype=np.int64)
        rs = np.array([b[1] for b in branches], dtype=np.int64)
        gs = np.array([b[2] for b in branches], dtype=np.int64)
        out = np.zeros((n, v.shape[1]))
        lse = np.zeros(n)
        st = self.lib.oracle_multibranch_f64(_ptr(q, _d), _ptr(k, _d), _ptr(v, _d), n, d, v.shape[1], len(branches),
                                             _ptr(ws, _i64p), _ptr(rs, _i64p), _ptr(gs, _i64p), int(scale),
                                             _ptr(out, _d), _ptr(lse, _d))
        if st:
            raise OracleError(st)
        return out, lse

    def dilated_batched(self, q, k, v, w, r, offsets, threads=None):
        """[B, N, h, d] (f64) -> [B, N, h, dv]: dilated_attention per (image, head)
        on `threads` host threads (default: all)."""
        q, k, v = (np.ascontiguousarray(x, dtype=np.float64) for x in (q, k, v))
        B, n, h, d = q.shape
        dv = v.shape[3]
        offs = np.asarray(offsets, dtype=np.int64)
        out = np.zeros((B, n, h, dv))
        st = self.lib.oracle_dilated_batched_f64(_ptr(q, _d), _ptr(k, _d), _ptr(v, _d), B, n, h, d, dv, w, r,
                                                 _ptr(offs, _i64p), threads or _threads(), _ptr(out, _d))
        if st:
            raise OracleError(st)
        return out

    def multibranch_batched(self, q, k, v, branches, threads=None):
        """branches: list of (w, r, offsets[h]).  Returns (out [B, N, h, dv], lse [B, h, N])."""
        q, k, v = (np.ascontiguousarray(x, dtype=np.float64) for x in (q, k, v))
        B, n, h, d = q.shape
        dv = v.shape[3]
        ws = np.array([b[0] for b in branches], dtype=np.int64)
        rs = np.array([b[1] for b in branches], dtype=np.int64)
        gs = np.ascontiguousarray(np.array([list(b[2]) for b in branches], dtype=np.int64))
        out = np.zeros((B, n, h, dv))
        lse = np.zeros((B, h, n))
        st = self.lib.oracle_multibranch_batched_f64(_ptr(q, _d), _ptr(k, _d), _ptr(v, _d), B, n, h, d, dv,
                                                     len(branches), _ptr(ws, _i64p), _ptr(rs, _i64p), _ptr(gs, _i64p),
                                                     threads or _threads(), _ptr(out, _d), _ptr(lse, _d))
        if st:
            raise OracleError(st)
        return out, lse

    def dilated_backward(self, q, k, v, do, w, r, gamma, scale=True):
        """Gradients (dq, dk, dv) of sum(O * do) for one head (f64)."""
        q, k, v, do = (np.ascontiguousarray(x, dtype=np.float64) for x in (q, k, v, do))
        n, d = q.shape
        dv = v.shape[1]
        gq, gk, gv = np.zeros((n, d)), np.zeros((n, d)), np.zeros((n, dv))
        st = self.lib.oracle_dilated_backward_f64(_ptr(q, _d), _ptr(k, _d), _ptr(v, _d), _ptr(do, _d), n, d, dv, w,
                                                  r, gamma, int(scale), _ptr(gq, _d), _ptr(gk, _d), _ptr(gv, _d))
        if st:
            raise OracleError(st)
        return gq, gk, gv

    def time_dilated_f32(self, q, k, v, w, r, units):
        """q, k, v: [distinct, N, d] float32.  Seconds for `units` forwards, 1 thread."""
        q, k, v = (np.ascontiguousarray(x, dtype=np.float32) for x in (q, k, v))
        distinct, n, d = q.shape
        out = np.zeros((n, d), dtype=np.float32)
        return self.lib.oracle_time_dilated_f32(_ptr(q, _f), _ptr(k, _f), _ptr(v, _f), n, w, r, d, units, distinct,
                                                _ptr(out, _f))


class Reference:
    """The unmodified reference behind ref_shim.cpp (oracle/_ref/libattnkit_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle ref; needs /root/reference)")
        self.lib = ctypes.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = ctypes.c_char_p
        for sfx, tp in (("f32", _f), ("f64", _d)):
            fn = getattr(L, f"ref_dilated_attention_{sfx}")
            fn.restype = _i32
            fn.argtypes = [tp, tp, tp, _i64, _i64, _i64, _i64, _i64, _i64, _i32, _i32, _i64, _i32, tp]
            fn = getattr(L, f"ref_naive_attention_{sfx}")
            fn.restype = _i32
            fn.argtypes = [tp, tp, tp, _i64, _i64, _i64, _i64, _i32, tp]
            fn = getattr(L, f"ref_randn_{sfx}")
            fn.restype = None
            fn.argtypes = [ctypes.c_uint64, _i64, tp]
        L.ref_masked_dense_dilated_f64.restype = _i32
        L.ref_masked_dense_dilated_f64.argtypes = [_d, _d, _d, _i64, _i64, _i64, _i64, _i64, _i64, _i32, _d]
        L.ref_segment_view.restype = _i32
        L.ref_segment_view.argtypes = [_i64, _i64, _i64, _i64, _i64, _i64p, _i64, _i64p]
        L.ref_validate.restype = _i32
        L.ref_validate.argtypes = [_i64, _i64, _i64, _i64, _i64, _i64p, _i64, _i32, _i64, _i32]
        L.ref_flop_count.restype = _i32
        L.ref_flop_count.argtypes = [_i64, _i64, _i64, _i64, _i64, _i64p, ctypes.POINTER(ctypes.c_uint64),
                                     ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_double),
                                     ctypes.c_char_p, _i64]
        L.ref_time_dilated_f32.restype = ctypes.c_double
        L.ref_time_dilated_f32.argtypes = [_i64, _i64, _i64, _i64, _i64, _i32, _i32, ctypes.c_uint64]
        L.ref_save_tensor.restype = _i32
        L.ref_save_tensor.argtypes = [ctypes.c_char_p, _i32, _i32, _i64p, ctypes.c_void_p]
        L.ref_load_tensor_f64.restype = _i32
        L.ref_load_tensor_f64.argtypes = [ctypes.c_char_p, _d, _i64, ctypes.POINTER(_i32), _i64p]
        for sfx, tp in (("f32", _f), ("f64", _d)):
            fn = getattr(L, f"ref_multi_head_dilated_{sfx}")
            fn.restype = _i32
            fn.argtypes = [tp, tp, tp, tp, tp, _i64, _i64, _i64, _i64, _i64, _i64p, tp]
        L.ref_dilated_backward_f64.restype = _i32
        L.ref_dilated_backward_f64.argtypes = [_d, _d, _d, _d, _i64, _i64, _i64, _i64, _i64, _i64, _d, _d, _d]
        L.ref_bench_csv_header.restype = _i32
        L.ref_bench_csv_header.argtypes = [ctypes.c_char_p, _i64]
        L.ref_spearman.restype = _i32
        L.ref_spearman.argtypes = [_d, _d, _i64, _d]
        L.ref_encoder_block_f64.restype = _i32
        L.ref_encoder_block_f64.argtypes = [_d, _i64, _i64, _i64, _i64, _i64, _i64] + [_d] * 14

    def last_error(self) -> str:
        return self.lib.ref_last_error().decode()

    def dilated_attention(self, q, k, v, w, r, gamma, scale=True, tiled=False, tile=1, workers=1):
        dt = q.dtype
        tp, fn = (_f, self.lib.ref_dilated_attention_f32) if dt == np.float32 else (
            _d, self.lib.ref_dilated_attention_f64)
        q, k, v = (np.ascontiguousarray(x, dtype=dt) for x in (q, k, v))
        n, d = q.shape
        out = np.zeros((n, v.shape[1]), dtype=dt)
        st = fn(_ptr(q, tp), _ptr(k, tp), _ptr(v, tp), n, d, v.shape[1], w, r, gamma, int(scale), int(tiled), tile,
                workers, _ptr(out, tp))
        if st:
            raise OracleError(st, self.last_error())
        return out

    def naive_attention(self, q, k, v, scale=True):
        dt = q.dtype
        tp, fn = (_f, self.lib.ref_naive_attention_f32) if dt == np.float32 else (_d, self.lib.ref_naive_attention_f64)
        q, k, v = (np.ascontiguousarray(x, dtype=dt) for x in (q, k, v))
        out = np.zeros((q.shape[0], v.shape[1]), dtype=dt)
        st = fn(_ptr(q, tp), _ptr(k, tp), _ptr(v, tp), q.shape[0], k.shape[0], q.shape[1], v.shape[1], int(scale),
                _ptr(out, tp))
        if st:
            raise OracleError(st, self.last_error())
        return out

    def masked_dense(self, q, k, v, w, r, gamma, scale=True):
        q, k, v = (np.ascontiguousarray(x, dtype=np.float64) for x in (q, k, v))
        n, d = q.shape
        out = np.zeros((n, v.shape[1]))
        st = self.lib.ref_masked_dense_dilated_f64(_ptr(q, _d), _ptr(k, _d), _ptr(v, _d), n, d, v.shape[1], w, r,
                                                   gamma, int(scale), _ptr(out, _d))
        if st:
            raise OracleError(st, self.last_error())
        return out

    def segment_view(self, n, w, r, i, g):
        cnt = ctypes.c_int64(0)
        buf = np.zeros(max(1, (w + r - 1) // r), dtype=np.int64)
        st = self.lib.ref_segment_view(n, w, r, i, g, _ptr(buf, _i64p), len(buf), ctypes.byref(cnt))
        if st:
            raise OracleError(st, self.last_error())
        return [int(x) for x in buf[: cnt.value]]

    def validate(self, n, w, r, h, d, offsets, tiled=False, tile=1, full=False):
        offs = np.asarray(offsets, dtype=np.int64)
        st = self.lib.ref_validate(n, w, r, h, d, _ptr(offs, _i64p), len(offs), int(tiled), tile, int(full))
        return st, (self.last_error() if st else "")

    def flop_count(self, n, w, r, h, d, offsets):
        offs = np.asarray(offsets, dtype=np.int64)
        a, b, c = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_double()
        buf = ctypes.create_string_buffer(256)
        st = self.lib.ref_flop_count(n, w, r, h, d, _ptr(offs, _i64p), ctypes.byref(a), ctypes.byref(b),
                                     ctypes.byref(c), buf, 256)
        if st:
            raise OracleError(st, self.last_error())
        return a.value, b.value, c.value, buf.value.decode()

    def randn(self, seed: int, n: int, dtype=np.float64):
        out = np.zeros(n, dtype=dtype)
        if dtype == np.float32:
            self.lib.ref_randn_f32(seed, n, _ptr(out, _f))
        else:
            self.lib.ref_randn_f64(seed, n, _ptr(out, _d))
        return out

    def time_dilated_f32(self, n, w, r, d, units, threads, distinct=8, seed=901):
        return self.lib.ref_time_dilated_f32(n, w, r, d, units, threads, distinct, seed)

    # ------------------------------------------------------------ §8(f) rows
    def save_tensor(self, path, array):
        a = np.asarray(array)
        a = np.asarray(a, dtype=np.float32 if a.dtype == np.float32 else np.float64, order="C")
        dims = np.array(a.shape, dtype=np.int64).reshape(-1)
        st = self.lib.ref_save_tensor(os.fsencode(path), 0 if a.dtype == np.float32 else 1, a.ndim,
                                      _ptr(dims, _i64p) if a.ndim else None, a.ctypes.data)
        if st:
            raise OracleError(st, self.last_error())

    def load_tensor(self, path, cap=1 << 24):
        out = np.zeros(cap)
        rank = ctypes.c_int32(0)
        dims = np.zeros(8, dtype=np.int64)
        st = self.lib.ref_load_tensor_f64(os.fsencode(path), _ptr(out, _d), cap, ctypes.byref(rank), _ptr(dims, _i64p))
        if st:
            raise OracleError(st, self.last_error())
        shape = tuple(int(x) for x in dims[: rank.value])
        return out[: int(np.prod(shape)) if shape else 1].reshape(shape)

    def multi_head_dilated(self, x, wq, wk, wv, wo, w, r, offsets=None):
        """x [N, D]; wq/wk/wv [h, D, d]; wo [D, D] (float32 or float64)."""
        dt = x.dtype
        tp, fn = (_f, self.lib.ref_multi_head_dilated_f32) if dt == np.float32 else (
            _d, self.lib.ref_multi_head_dilated_f64)
        x, wq, wk, wv, wo = (np.ascontiguousarray(a, dtype=dt) for a in (x, wq, wk, wv, wo))
        n, dm = x.shape
        h = wq.shape[0]
        offs = np.asarray(offsets if offsets is not None else [j % r for j in range(h)], dtype=np.int64)
        out = np.zeros((n, dm), dtype=dt)
        st = fn(_ptr(x, tp), _ptr(wq, tp), _ptr(wk, tp), _ptr(wv, tp), _ptr(wo, tp), n, dm, h, w, r,
                _ptr(offs, _i64p), _ptr(out, tp))
        if st:
            raise OracleError(st, self.last_error())
        return out

    def dilated_backward(self, q, k, v, do, w, r, gamma):
        q, k, v, do = (np.ascontiguousarray(a, dtype=np.float64) for a in (q, k, v, do))
        n, d = q.shape
        dv = v.shape[1]
        gq, gk, gv = np.zeros((n, d)), np.zeros((n, d)), np.zeros((n, dv))
        st = self.lib.ref_dilated_backward_f64(_ptr(q, _d), _ptr(k, _d), _ptr(v, _d), _ptr(do, _d), n, d, dv, w, r,
                                               gamma, _ptr(gq, _d), _ptr(gk, _d), _ptr(gv, _d))
        if st:
            raise OracleError(st, self.last_error())
        return gq, gk, gv

    def bench_csv_header(self) -> str:
        buf = ctypes.create_string_buffer(512)
        st = self.lib.ref_bench_csv_header(buf, 512)
        if st:
            raise OracleError(st, self.last_error())
        return buf.value.decode()

    def spearman(self, a, b) -> float:
        a, b = (np.ascontiguousarray(x, dtype=np.float64) for x in (a, b))
        out = ctypes.c_double(0)
        st = self.lib.ref_spearman(_ptr(a, _d), _ptr(b, _d), len(a), ctypes.byref(out))
        if st:
            raise OracleError(st, self.last_error())
        return out.value

    def encoder_block(self, x, p, h, w, r):
        """One pre-norm block (encoder.hpp:241-248).  p: dict with ln1_g, ln1_b,
        wq, wk, wv [h, D, d], wo, bo, ln2_g, ln2_b, w1, b1, w2, b2."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        n, dm = x.shape
        hidden = p["w1"].shape[1]
        keys = ["ln1_g", "ln1_b", "wq", "wk", "wv", "wo", "bo", "ln2_g", "ln2_b", "w1", "b1", "w2", "b2"]
        arrs = [np.ascontiguousarray(p[k], dtype=np.float64) for k in keys]
        out = np.zeros((n, dm))
        st = self.lib.ref_encoder_block_f64(_ptr(x, _d), n, dm, h, hidden, w, r, *[_ptr(a, _d) for a in arrs],
                                            _ptr(out, _d))
        if st:
            raise OracleError(st, self.last_error())
        return out


def reference_available() -> bool:
    return os.path.exists(REF_SO)
