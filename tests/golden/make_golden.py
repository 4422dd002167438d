#!/usr/bin/env python3
"""Regenerate tests/golden/ from the UNMODIFIED reference (oracle/_ref).

The reference ships no on-disk fixtures (its tests draw inputs from a seeded
mt19937_64); these vectors pin its outputs.  Inputs come from numpy PCG64 with
the listed seeds (reproducible on any host); outputs are
attnkit::dilated_attention<double|float> run through oracle/_ref/
libattnkit_ref.so, which `make -C oracle ref` builds from /root/reference.
Run from the repo root:  python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Reference  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# (N, w, r, gamma, d, dv, tiled, tile, scale): the reference's test geometries
# (test_attention.cpp / acceptance.cpp) plus tails and d != dv.
CASES = [
    (8, 4, 2, 0, 4, 4, 0, 1, 1), (8, 4, 2, 1, 4, 4, 0, 1, 1), (16, 4, 2, 1, 4, 4, 0, 1, 1),
    (10, 4, 2, 1, 4, 4, 0, 1, 1), (12, 12, 1, 0, 4, 4, 0, 1, 1), (32, 8, 4, 3, 8, 8, 0, 1, 1),
    (64, 16, 2, 1, 8, 8, 0, 1, 1), (32, 16, 2, 0, 8, 8, 1, 2, 1), (33, 7, 3, 2, 8, 5, 0, 1, 1),
    (100, 30, 4, 3, 16, 16, 0, 1, 1), (16, 8, 2, 1, 4, 4, 0, 1, 0), (40, 9, 4, 2, 8, 8, 1, 3, 1),
    (256, 64, 2, 1, 16, 16, 0, 1, 1), (257, 64, 4, 3, 16, 16, 0, 1, 1),
]


def main():
    ref = Reference()
    arrays, meta = {}, []
    for i, (n, w, r, g, d, dv, tiled, tile, scale) in enumerate(CASES):
        rng = np.random.default_rng(1000 + i)
        q, k = rng.standard_normal((n, d)), rng.standard_normal((n, d))
        v = rng.standard_normal((n, dv))
        out = ref.dilated_attention(q, k, v, w, r, g, scale=bool(scale), tiled=bool(tiled), tile=tile)
        arrays.update({f"q{i}": q, f"k{i}": k, f"v{i}": v, f"o{i}": out})
        meta.append(dict(N=n, w=w, r=r, gamma=g, d=d, dv=dv, tiled=tiled, tile=tile, scale=scale, seed=1000 + i))
    np.savez_compressed(os.path.join(HERE, "dilated_small.npz"), **arrays)

    # Headline (config 1): N=4096, w=512, r=2, d=64, gamma=0, float32.
    rng = np.random.default_rng(901)
    q, k, v = (rng.standard_normal((4096, 64)).astype(np.float32) for _ in range(3))
    out = ref.dilated_attention(q, k, v, 512, 2, 0)
    rows = list(range(0, 4096, 256))
    headline = dict(N=4096, w=512, r=2, gamma=0, d=64, dtype="float32", input_seed=901,
                    input_draw="np.random.default_rng(901).standard_normal((4096, 64)).astype(float32) for q, k, v",
                    sha256=hashlib.sha256(out.tobytes()).hexdigest(), sample_rows=rows,
                    sample=out[rows].tolist(), checksum=float(out.astype(np.float64).sum()))
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py via oracle/_ref (unmodified reference)",
                   "small_cases": meta, "headline_f32": headline}, f, indent=1)
    print(f"wrote {len(CASES)} small cases + headline")


if __name__ == "__main__":
    main()
