"""Committed golden vectors (tests/golden/, generated from the unmodified
reference by make_golden.py): the oracle port must reproduce them bit for
bit; on the GPU the device kernels must match them within tolerance."""
import hashlib
import json
import os

import numpy as np
import pytest

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load():
    meta = json.load(open(os.path.join(HERE, "golden.json")))
    arrs = np.load(os.path.join(HERE, "dilated_small.npz"))
    return meta, arrs


def test_port_reproduces_golden_small(port):
    meta, arrs = load()
    for i, c in enumerate(meta["small_cases"]):
        got = port.dilated_attention(arrs[f"q{i}"], arrs[f"k{i}"], arrs[f"v{i}"], c["w"], c["r"], c["gamma"],
                                     scale=bool(c["scale"]), tiled=bool(c["tiled"]), tile=c["tile"])
        assert got.tobytes() == arrs[f"o{i}"].tobytes(), c


def test_port_reproduces_golden_headline(port):
    h = json.load(open(os.path.join(HERE, "golden.json")))["headline_f32"]
    rng = np.random.default_rng(h["input_seed"])
    q, k, v = (rng.standard_normal((4096, 64)).astype(np.float32) for _ in range(3))
    out = port.dilated_attention(q, k, v, h["w"], h["r"], h["gamma"])
    assert np.array_equal(out[h["sample_rows"]], np.array(h["sample"], dtype=np.float32))
    assert hashlib.sha256(out.tobytes()).hexdigest() == h["sha256"]


@pytest.mark.gpu
def test_device_matches_golden(dfa, cuda):
    import torch

    meta, arrs = load()
    for i, c in enumerate(meta["small_cases"]):
        cfg = dfa.AttentionConfig(c["N"], c["w"], c["r"], 1, c["d"], [c["gamma"]],
                                  "tiled" if c["tiled"] else "naive", c["tile"], bool(c["scale"]))
        q, k, v = (torch.from_numpy(arrs[f"{n}{i}"]).float().cuda() for n in "qkv")
        got = dfa.dilated_attention(q, k, v, cfg, c["gamma"]).double().cpu().numpy()
        assert np.abs(got - arrs[f"o{i}"]).max() <= 1e-4, c
    h = meta["headline_f32"]
    rng = np.random.default_rng(h["input_seed"])
    q, k, v = (torch.from_numpy(rng.standard_normal((4096, 64)).astype(np.float32)).cuda() for _ in range(3))
    cfg = dfa.AttentionConfig(4096, 512, 2, 1, 64, [0])
    got = dfa.dilated_attention(q, k, v, cfg, 0).cpu().numpy()
    assert np.abs(got[h["sample_rows"]] - np.array(h["sample"])).max() <= 1e-4
    assert abs(float(got.astype(np.float64).sum()) - h["checksum"]) <= 1e-4 * 4096 * 64
