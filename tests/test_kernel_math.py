"""Host restatements of the device-side arithmetic tricks (CPU)."""
import numpy as np


def ex2_poly(x):
    """float32 mirror of ptx::ex2_poly (sm100_ptx.cuh)."""
    x = np.maximum(x.astype(np.float32), np.float32(-125.0))
    magic = np.float32(12582912.0)
    t = (x + magic).astype(np.float32)
    f = (x - (t - magic)).astype(np.float32)
    p = np.float32(5.459282631e-2) * f + np.float32(2.422181094e-1)
    p = (p * f + np.float32(6.933686450e-1)).astype(np.float32)
    p = (p * f + np.float32(1.0)).astype(np.float32)
    bits = p.view(np.int32) + (t.view(np.int32) << 23)
    return bits.view(np.float32)


def test_ex2_poly_accuracy():
    x = np.linspace(-120, 8, 2_000_001, dtype=np.float32)
    got = ex2_poly(x).astype(np.float64)
    rel = np.abs(got / np.exp2(x.astype(np.float64)) - 1)
    assert rel.max() < 2e-4  # bf16 P carries 2^-9 = 2e-3 relative rounding anyway
    assert ex2_poly(np.array([0.0], np.float32))[0] == 1.0
    assert ex2_poly(np.array([-np.inf], np.float32))[0] < 1e-37


def fastdiv(n, d):
    """mirror of FastDiv (dfa_sm100.cu): q = (umulhi(n, mul) + n) >> shift."""
    shift = 0
    while (1 << shift) < d:
        shift += 1
    mul = 0 if d == 1 else (((1 << 32) * ((1 << shift) - d)) // d + 1) & 0xFFFFFFFF
    return ((n * mul >> 32) + n) >> shift


def test_fastdiv_exact():
    rng = np.random.default_rng(0)
    for d in [1, 2, 3, 5, 6, 7, 8, 16, 96, 128, 171, 256, 1000, 2048, 65535, 123457]:
        ns = list(rng.integers(0, 2**31 - 1, 2000)) + [0, 1, d - 1, d, d + 1, 2**31 - 1]
        for n in ns:
            assert fastdiv(int(n), d) == int(n) // d, (n, d)
