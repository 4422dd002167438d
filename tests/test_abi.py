"""The C-ABI library loads, exports every symbol include/dfa.h declares, and
its host-side entry points agree with the reference (CPU only, no launches)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "dfa.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(dfa_[a-z_0-9]+)\s*\(", src, flags=re.M)))


def test_header_declares_expected_entry_points():
    from paper_2403_09195_b200 import _lib

    assert header_functions() == sorted(_lib.EXPORTED)


def test_library_exports_every_declared_symbol():
    from paper_2403_09195_b200 import _lib

    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [f for f in header_functions() if f not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for f in header_functions():
        assert getattr(lib, f) is not None


def test_version_and_fault_flag(dfa):
    assert dfa.lib.dfa_version() >= 100
    assert dfa.lib.dfa_get_fault_perturb() == 0
    with dfa.fault_perturb():
        assert dfa.lib.dfa_get_fault_perturb() == 1
    assert dfa.lib.dfa_get_fault_perturb() == 0


def test_library_has_sm100a_code():
    """The shipped .so carries sm_100a SASS with tcgen05 and TMA instructions."""
    from paper_2403_09195_b200 import _lib

    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    if not sass:
        pytest.skip("cuobjdump unavailable")
    assert "UTCHMMA" in sass  # tcgen05.mma
    assert "UTMALDG" in sass  # TMA load
    assert "LDTM" in sass  # tcgen05.ld
    assert "arch = sm_100a" in subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True,
                                              text=True).stdout or "sm_100a" in sass


def test_query_path_dispatch(dfa):
    head = dfa.AttentionConfig(4096, 512, 2, 6, 64, [0, 1, 0, 1, 0, 1])
    assert dfa.query_path(head, "bf16", 64) == 1  # tcgen05
    assert dfa.query_path(head, "f32", 1) == 2  # fp32 validation mode -> SIMT
    assert dfa.query_path(dfa.AttentionConfig(10, 4, 3, 1, 64, [0]), "bf16", 1) == 2  # r !| N
    assert dfa.query_path(dfa.AttentionConfig(64, 16, 2, 1, 32, [0]), "bf16", 1) == 2  # d != 64


def test_unsupported_sizes_fail_loudly(dfa):
    with pytest.raises(dfa.UnsupportedError):
        dfa.query_path(dfa.AttentionConfig(64, 16, 2, 1, 512, [0]), "f32", 1)
    with pytest.raises(dfa.UnsupportedError):
        dfa.query_path(dfa.AttentionConfig(64, 16, 1, 300, 8, [0] * 300), "f32", 1)


def test_workspace_bytes(dfa):
    cfg = dfa.AttentionConfig(4096, 512, 2, 6, 64, [0, 1, 0, 1, 0, 1])
    n = dfa.Workspace.bytes_for(cfg, "bf16", 2)
    assert n == 4 * 2 * 4096 * 6 * 64 * 2


def test_entry_points_validate_before_touching_memory(dfa):
    """Every C-ABI entry validates geometry / sizes / workspaces and returns the
    reference-mapped status before any device access (fake pointers here)."""
    import ctypes

    from paper_2403_09195_b200 import _lib

    L = dfa.lib
    cfg = dfa.AttentionConfig(4096, 512, 2, 6, 64, [0, 1, 0, 1, 0, 1])
    c = cfg._c()
    fake = ctypes.c_void_p(0x1000)
    # token strides below h*d
    assert L.dfa_forward_strided(ctypes.byref(c), 1, 1, fake, 10, fake, 384, fake, 384, fake, 384, None,
                                 None) == _lib.DFA_ERR_DIMENSION
    # backward workspace too small
    assert L.dfa_backward(ctypes.byref(c), 1, 1, *([fake] * 10), 16, None) == _lib.DFA_ERR_DIMENSION
    # multibranch: 9 branches is over the limit
    br = (_lib.DfaBranch * 9)()
    need = ctypes.c_size_t(0)
    assert L.dfa_multibranch_workspace_bytes(ctypes.byref(c), 9, 1, 1, ctypes.byref(need)) == _lib.DFA_ERR_CONFIG
    assert L.dfa_forward_multibranch(ctypes.byref(c), 9, br, 1, 1, fake, fake, fake, fake, None, fake, 1 << 40,
                                     None) == _lib.DFA_ERR_CONFIG
    # multi-head needs full coverage; encoder block needs a positive MLP width
    partial = dfa.AttentionConfig(4096, 512, 4, 2, 64, [0, 1])._c()
    assert L.dfa_multi_head_workspace_bytes(ctypes.byref(partial), 1, 1, ctypes.byref(need)) == _lib.DFA_ERR_CONFIG
    assert "covered by no head" in L.dfa_last_error().decode()
    assert L.dfa_encoder_block_workspace_bytes(ctypes.byref(c), 1, 1, 0, ctypes.byref(need)) == _lib.DFA_ERR_CONFIG
    # bad dtype code
    assert L.dfa_forward(ctypes.byref(c), 7, 1, fake, fake, fake, fake, None, None) == _lib.DFA_ERR_CONFIG
    # batch 0 is a no-op success
    assert L.dfa_forward(ctypes.byref(c), 1, 0, fake, fake, fake, fake, None, None) == _lib.DFA_OK
    # null tensor pointers
    assert L.dfa_forward(ctypes.byref(c), 1, 1, None, fake, fake, fake, None, None) == _lib.DFA_ERR_DIMENSION


def test_host_transfer_bytes_for_pageable_memory(dfa):
    """Pageable host buffers cannot be read in place: the whole tensors are copied."""
    import torch

    cfg = dfa.AttentionConfig(1024, 256, 2, 2, 64, [0, 1])
    q, k, v = (torch.zeros((2, 1024, 2, 64), dtype=torch.bfloat16) for _ in range(3))
    h2d, d2h = dfa.host_transfer_bytes(q, k, v, cfg)
    assert (h2d, d2h) == (3 * q.numel() * 2, q.numel() * 2)
