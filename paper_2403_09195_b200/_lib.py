"""ctypes binding of the C-ABI in include/dfa.h (libdfa.so, built in-tree).

There is no fallback: if libdfa.so is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdfa.so")
# Profiling only: scripts/variants.py times alternative builds of the same
# sources (compile-time tuning knobs) by pointing this at another in-tree .so.
LIB_PATH = os.environ.get("DFA_LIB_VARIANT", LIB_PATH)

DFA_OK = 0
DFA_ERR_CONFIG = 1
DFA_ERR_DIMENSION = 2
DFA_ERR_OUT_OF_RANGE = 3
DFA_ERR_CONTRACT = 4
DFA_ERR_CUDA = 5
DFA_ERR_UNSUPPORTED = 6
DFA_ERR_IO = 7

DFA_F32 = 0
DFA_BF16 = 1
DFA_F64 = 2

DFA_PATH_NONE = 0
DFA_PATH_SM100_TCGEN05 = 1
DFA_PATH_SIMT = 2
DFA_MB_AUTO = 0
DFA_MB_PER_BRANCH = 1

# Every function include/dfa.h declares (tests check the .so exports them).
EXPORTED = (
    "dfa_last_error",
    "dfa_validate",
    "dfa_segment_view",
    "dfa_flop_count",
    "dfa_query_path",
    "dfa_forward",
    "dfa_workspace_create",
    "dfa_workspace_destroy",
    "dfa_dilated_attention_host",
    "dfa_forward_host",
    "dfa_forward_strided",
    "dfa_set_host_zero_copy",
    "dfa_set_host_kept_out",
    "dfa_host_transfer_bytes",
    "dfa_set_fault_perturb",
    "dfa_get_fault_perturb",
    "dfa_workspace_bytes",
    "dfa_set_path_override",
    "dfa_set_multibranch_mode",
    "dfa_set_multibranch_trace",
    "dfa_multibranch_plan",
    "dfa_forward_traced",
    "dfa_forward_debug",
    "dfa_multibranch_workspace_bytes",
    "dfa_forward_multibranch",
    "dfa_last_launch_count",
    "dfa_version",
    "dfa_backward_workspace_bytes",
    "dfa_backward",
    "dfa_multi_head_workspace_bytes",
    "dfa_multi_head_dilated",
    "dfa_multi_head_host_workspace_bytes",
    "dfa_multi_head_dilated_host",
    "dfa_encoder_block_workspace_bytes",
    "dfa_encoder_block_forward",
    "dfa_tensor_header",
    "dfa_tensor_load",
    "dfa_tensor_save",
    "dfa_gemm",
    "dfa_set_gemm_tile",
)


class DfaBlockWeights(ctypes.Structure):
    """Mirror of dfa_block_weights_t (include/dfa.h)."""

    _fields_ = [(n, ctypes.c_void_p) for n in ("ln1_g", "ln1_b", "wq", "wk", "wv", "wo", "bo", "ln2_g", "ln2_b", "w1",
                                                "b1", "w2", "b2")] + [("hidden", ctypes.c_int64)]


class DfaConfig(ctypes.Structure):
    """Mirror of dfa_config_t (include/dfa.h)."""

    _fields_ = [
        ("seq_len", ctypes.c_int64),
        ("segment_len", ctypes.c_int64),
        ("interval", ctypes.c_int64),
        ("num_heads", ctypes.c_int64),
        ("head_dim", ctypes.c_int64),
        ("value_dim", ctypes.c_int64),
        ("head_offsets", ctypes.POINTER(ctypes.c_int64)),
        ("kernel", ctypes.c_int32),
        ("tile_size", ctypes.c_int64),
        ("scale_scores", ctypes.c_int32),
    ]


class DfaBranch(ctypes.Structure):
    """Mirror of dfa_branch_t (include/dfa.h)."""

    _fields_ = [
        ("segment_len", ctypes.c_int64),
        ("interval", ctypes.c_int64),
        ("head_offsets", ctypes.POINTER(ctypes.c_int64)),
    ]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C paper_2403_09195_b200/csrc` "
            "(or __graft_entry__.build()); there is no CPU fallback"
        )
    lib = ctypes.CDLL(LIB_PATH)
    c_i64, c_i32, c_vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
    p_cfg = ctypes.POINTER(DfaConfig)
    p_i64 = ctypes.POINTER(ctypes.c_int64)
    sig = {
        "dfa_last_error": (ctypes.c_char_p, []),
        "dfa_validate": (c_i32, [p_cfg, c_i32]),
        "dfa_segment_view": (c_i32, [c_i64, c_i64, c_i64, c_i64, c_i64, p_i64, c_i64, p_i64]),
        "dfa_flop_count": (
            c_i32,
            [p_cfg, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_double)],
        ),
        "dfa_query_path": (c_i32, [p_cfg, c_i32, c_i64, ctypes.POINTER(c_i32)]),
        "dfa_forward": (c_i32, [p_cfg, c_i32, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
        "dfa_workspace_create": (c_i32, [ctypes.c_size_t, ctypes.POINTER(c_vp)]),
        "dfa_workspace_destroy": (c_i32, [c_vp]),
        "dfa_dilated_attention_host": (c_i32, [p_cfg, c_i32, c_vp, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp]),
        "dfa_forward_host": (c_i32, [p_cfg, c_i32, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
        "dfa_set_fault_perturb": (None, [c_i32]),
        "dfa_get_fault_perturb": (c_i32, []),
        "dfa_workspace_bytes": (c_i32, [p_cfg, c_i32, c_i64, c_i32, ctypes.POINTER(ctypes.c_size_t)]),
        "dfa_set_path_override": (None, [c_i32]),
        "dfa_set_multibranch_mode": (None, [c_i32]),
        "dfa_set_multibranch_trace": (None, [c_vp]),
        "dfa_multibranch_plan": (c_i32, [p_cfg, c_i32, ctypes.POINTER(DfaBranch), c_i64, c_i32, c_vp, ctypes.c_size_t,
                                         ctypes.POINTER(c_i32), ctypes.POINTER(c_i32), ctypes.POINTER(c_i32),
                                         ctypes.POINTER(c_i32)]),
        "dfa_forward_traced": (c_i32, [p_cfg, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
        "dfa_forward_debug": (c_i32, [p_cfg, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
        "dfa_multibranch_workspace_bytes": (c_i32, [p_cfg, c_i32, c_i32, c_i64, ctypes.POINTER(ctypes.c_size_t)]),
        "dfa_forward_multibranch": (c_i32, [p_cfg, c_i32, ctypes.POINTER(DfaBranch), c_i32, c_i64, c_vp, c_vp, c_vp,
                                            c_vp, c_vp, c_vp, ctypes.c_size_t, c_vp]),
        "dfa_last_launch_count": (c_i32, []),
        "dfa_version": (c_i32, []),
        "dfa_backward_workspace_bytes": (c_i32, [p_cfg, c_i64, ctypes.POINTER(ctypes.c_size_t)]),
        "dfa_backward": (c_i32, [p_cfg, c_i32, c_i64] + [c_vp] * 10 + [ctypes.c_size_t, c_vp]),
        "dfa_multi_head_workspace_bytes": (c_i32, [p_cfg, c_i32, c_i64, ctypes.POINTER(ctypes.c_size_t)]),
        "dfa_multi_head_dilated": (c_i32, [p_cfg, c_i32, c_i64] + [c_vp] * 7 + [ctypes.c_size_t, c_vp]),
        "dfa_multi_head_host_workspace_bytes": (c_i32, [p_cfg, c_i32, c_i64, ctypes.POINTER(ctypes.c_size_t)]),
        "dfa_multi_head_dilated_host": (c_i32, [p_cfg, c_i32, c_i64] + [c_vp] * 7),
        "dfa_encoder_block_workspace_bytes": (c_i32, [p_cfg, c_i32, c_i64, c_i64, ctypes.POINTER(ctypes.c_size_t)]),
        "dfa_encoder_block_forward": (c_i32, [p_cfg, c_i32, c_i64, c_vp, ctypes.POINTER(DfaBlockWeights), c_vp, c_vp,
                                              ctypes.c_size_t, c_vp]),
        "dfa_forward_strided": (c_i32, [p_cfg, c_i32, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64,
                                        c_vp, c_vp]),
        "dfa_set_host_zero_copy": (None, [c_i32]),
        "dfa_set_host_kept_out": (None, [c_i32]),
        "dfa_host_transfer_bytes": (c_i32, [p_cfg, c_i32, c_i64, c_vp, c_vp, c_vp, c_vp, c_i32,
                                            ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(ctypes.c_size_t)]),
        "dfa_tensor_header": (c_i32, [ctypes.c_char_p, ctypes.POINTER(c_i32), ctypes.POINTER(c_i32), p_i64]),
        "dfa_tensor_load": (c_i32, [ctypes.c_char_p, c_i32, c_vp, c_i64]),
        "dfa_tensor_save": (c_i32, [ctypes.c_char_p, c_i32, c_i32, p_i64, c_vp]),
        "dfa_set_gemm_tile": (None, [c_i32]),
        "dfa_gemm": (c_i32, [c_i32, c_i64, c_i64, c_i64, c_i64, c_vp, c_i64, c_i64, c_vp, c_i64, c_i64, c_vp, c_i64,
                             c_i64, c_vp, c_i64, ctypes.c_float, c_vp, c_i32, c_vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()
