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
