"""include/dfa.hpp used from C++ the way the reference is (compiled with g++,
linked against libdfa.so)."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def binary(tmp_path_factory):
    from paper_2403_09195_b200 import _lib

    out = tmp_path_factory.mktemp("cpp") / "dfa_hpp_check"
    libdir = os.path.dirname(_lib.LIB_PATH)
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "dfa_hpp_check.cpp"), "-L", libdir, "-ldfa",
                    f"-Wl,-rpath,{libdir}", "-o", str(out)], check=True)
    return str(out)


def test_cpp_host_api(binary):
    r = subprocess.run([binary], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_dilated_attention_on_gpu(binary, port, tmp_path):
    r = subprocess.run([binary, "gpu", str(tmp_path)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    q, k, v, o = (np.fromfile(tmp_path / f"{n}.f32", dtype=np.float32).reshape(4096, 64) for n in "qkvo")
    want = port.dilated_attention(q.astype(np.float64), k.astype(np.float64), v.astype(np.float64), 512, 2, 1)
    assert np.abs(o - want).max() <= 1e-4


@pytest.mark.gpu
def test_cpp_multi_head_dilated_vs_reference(binary, ref, tmp_path):
    """dfa::multi_head_dilated (C++ adapter over dfa_multi_head_dilated_host)
    vs the compiled reference's multi_head_dilated on the same fp32 inputs."""
    r = subprocess.run([binary, "gpu", str(tmp_path)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    ld = lambda n, shape: np.fromfile(tmp_path / f"{n}.f32", dtype=np.float32).reshape(shape)  # noqa: E731
    x, wo, y = ld("mh_x", (256, 128)), ld("mh_wo", (128, 128)), ld("mh_y", (256, 128))
    wq, wk, wv = (np.stack([ld(f"mh_{n}{j}", (128, 64)) for j in range(2)]) for n in ("wq", "wk", "wv"))
    want = ref.multi_head_dilated(x, wq, wk, wv, wo, 64, 2)
    assert np.abs(y - want).max() <= 1e-4 * max(1.0, np.abs(want).max())


@pytest.mark.gpu
def test_reference_acceptance_gates_through_dfa_hpp(binary):
    """The reference's acceptance gates 1 (masked oracle, f64, 1e-10), 3
    (collapse, f32, 1e-6) and 8 (worker determinism, f64, bitwise) with the
    reference's seeds and draws, every dilated_attention call going through
    dfa::dilated_attention (float -> fp32 kernel, double -> f64 kernel)."""
    r = subprocess.run([binary, "gates"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    for gate in (1, 3, 8):
        assert f"GATE {gate} " in r.stdout and "FAIL" not in r.stdout, r.stdout
