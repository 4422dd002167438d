"""DTNSR1 tensor files (tensor_io.hpp:15-19, 52-156): the C-ABI reader/writer
(dfa_tensor_*) against the compiled reference's save_tensor / load_tensor --
files written by either side load bit-exactly on the other -- and the
reference's malformed-input cases (test_tensor.cpp:209-221) with its io_error
text.  CPU only."""
import os

import numpy as np
import pytest


@pytest.mark.parametrize("shape", [(3, 4, 2), (5,), (), (1, 1, 1, 1, 1, 1, 1, 1), (0, 3)])
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_roundtrip_and_reference_compat(dfa, ref, tmp_path, shape, dt):
    a = np.random.default_rng(7).standard_normal(shape).astype(dt)
    ours, theirs = str(tmp_path / "ours.tnsr"), str(tmp_path / "ref.tnsr")
    dfa.save_tensor(ours, a)
    ref.save_tensor(theirs, a)
    assert open(ours, "rb").read() == open(theirs, "rb").read()  # byte-identical files
    want_dt = "f32" if dt == np.float32 else "f64"
    assert dfa.tensor_header(theirs) == (want_dt, shape)
    b = dfa.load_tensor(theirs, want_dt)
    assert b.shape == shape and b.dtype == dt and np.array_equal(a, b)
    c = ref.load_tensor(ours)
    assert c.shape == shape and np.array_equal(a.astype(np.float64), c)


def test_dtype_conversion_like_read_payload(dfa, tmp_path):
    """test_tensor.cpp:200-206: an f64 payload read into an f32 pipeline converts."""
    d = np.random.default_rng(1).standard_normal(5)
    p = str(tmp_path / "d.tnsr")
    dfa.save_tensor(p, d)
    f = dfa.load_tensor(p, "f32")
    assert f.dtype == np.float32 and np.allclose(f, d, rtol=1e-6)
    f32 = d.astype(np.float32)
    dfa.save_tensor(p, f32)
    assert np.array_equal(dfa.load_tensor(p, "f64"), f32.astype(np.float64))


def test_malformed_files_raise_io_error(dfa, ref, tmp_path):
    """test_tensor.cpp:209-221 -- same cases, same error class (io_error) and text."""
    from oracle.oracle import OracleError

    bad_magic = tmp_path / "bad_magic.tnsr"
    bad_magic.write_bytes(b"XXXXXXxxxxxxxx")
    full = tmp_path / "full.tnsr"
    dfa.save_tensor(str(full), np.ones((4, 4), dtype=np.float32))
    cut = tmp_path / "cut.tnsr"
    cut.write_bytes(full.read_bytes()[:-5])
    bad_dtype = tmp_path / "bad_dtype.tnsr"
    bad_dtype.write_bytes(b"DTNSR1" + bytes([9, 1]))
    big_rank = tmp_path / "big_rank.tnsr"
    big_rank.write_bytes(b"DTNSR1" + bytes([0, 9]))
    for path in (bad_magic, cut, bad_dtype, big_rank):
        with pytest.raises(dfa.TensorIOError) as ours:
            dfa.load_tensor(str(path), "f32")
        with pytest.raises(OracleError) as theirs:
            ref.load_tensor(str(path))
        assert theirs.value.code == 7  # io_error
        assert str(ours.value) in str(theirs.value), (str(ours.value), str(theirs.value))
    with pytest.raises(dfa.TensorIOError, match="cannot open tensor file"):
        dfa.load_tensor(str(tmp_path / "missing.tnsr"))
    with pytest.raises(dfa.TensorIOError, match="exceeds format limit"):
        dfa.save_tensor(str(tmp_path / "r9.tnsr"), np.zeros((1,) * 9))
    assert not os.path.exists(str(tmp_path / "r9.tnsr"))
