"""The tcgen05 kernel's mbarrier protocol, executed as a model (CPU).

scripts/protocol_model.py mirrors every role loop of dfa_sm100_kernel and
checks, under several interleavings, that no CTA deadlocks and that every
parity wait sees its barrier at most one phase away (the hardware parity
check is ambiguous otherwise).  A round-1 bug -- the softmax publishing row
statistics two units ahead of the epilogue when m <= 128 -- was found this way
and is pinned by test_model_flags_the_stat_full_hazard."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import protocol_model as pm  # noqa: E402

GEOMS = [(4096, w, r) for w in (256, 512, 1024, 2048, 4096) for r in (1, 2, 4, 8)] + [
    (1000, 300, 2), (512, 64, 2), (768, 96, 1), (640, 640, 1), (4104, 513, 3), (130, 130, 2), (1024, 256, 2)]


@pytest.mark.parametrize("n,w,r", GEOMS)
def test_protocol_is_deadlock_and_parity_safe(n, w, r):
    for B, h, grid in ((3, 6, 148), (2, 2, 7), (1, 1, 3)):
        p = pm.params(n, w, r, h, B, grid)
        for cta in range(min(grid, p["n_units"])):
            for seed in (0, 1, 2):
                assert pm.run(p, cta, seed) is None, (n, w, r, B, h, grid, cta, seed)


def test_model_flags_the_stat_full_hazard(monkeypatch):
    """Without the stat_empty handshake the model reports the parity hazard."""
    def softmax_without_handshake(p, B, cta, s):
        gen = orig(p, B, cta, s)
        item = next(gen, None)
        while item is not None:
            if item[1].name.startswith("stat_empty"):
                item = next(gen, None)  # skip the wait
                continue
            yield item
            item = next(gen, None)

    orig = pm.softmax
    monkeypatch.setattr(pm, "softmax", softmax_without_handshake)
    p = pm.params(4096, 256, 2, 6, 64, 148)
    with pytest.raises(pm.ParityHazard):
        for seed in range(3):
            pm.run(p, 10, seed)
