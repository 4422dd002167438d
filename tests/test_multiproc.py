"""Batch sharding + final gather with world_size 2 on gloo (CPU)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_09195_b200.dist import gather_to_rank0, shard_range, shard_sizes


def test_shard_ranges_cover_exactly():
    for total in (0, 1, 7, 64, 8192, 8193):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                a, b = shard_range(total, r, world)
                seen.extend(range(a, b))
            assert seen == list(range(total))
            sizes = shard_sizes(total, world)
            assert max(sizes) - min(sizes) <= 1
    assert shard_sizes(8192, 8) == [1024] * 8
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, total, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = shard_range(total, rank, world)
    # stand-in for each rank's dfa_forward output: image index in every element
    shard = torch.arange(a, b, dtype=torch.float32).view(-1, 1, 1).expand(-1, 3, 2).contiguous()
    out = gather_to_rank0(shard, total)
    if rank == 0:
        q.put(out.numpy().tolist())
    else:
        assert out is None
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [8, 9, 64])
def test_gather_world2_gloo(total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    t = torch.tensor(got)
    assert t.shape == (total, 3, 2)
    assert torch.equal(t[:, 0, 0], torch.arange(total, dtype=torch.float32))


def test_segment_shards_cover_whole_segments():
    from paper_2403_09195_b200.dist import segment_shard

    for n, w in ((4096, 512), (4096, 4096), (1000, 300), (130, 64)):
        for world in (1, 2, 3, 4, 8):
            rows = []
            for r in range(world):
                a, b = segment_shard(n, w, r, world)
                assert a == b or (a % w == 0 and (b % w == 0 or b == n))  # whole segments only
                rows.extend(range(a, b))
            assert rows == list(range(n))


def _seg_worker(rank, world, port, q):
    """segment_parallel_forward's plumbing on gloo with a CPU stand-in for the
    kernel (the real one needs a GPU): each rank "computes" its rows and the
    all-gather must reassemble the full sequence in order."""
    import dataclasses

    import paper_2403_09195_b200 as dfa_pkg
    from paper_2403_09195_b200 import dist as ddist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def fake_forward(qq, kk, vv, cfg, out=None, stream=None):
        assert qq.shape[1] == cfg.seq_len  # the local problem keeps the segment grid
        cfg.validate()  # a tail-only shard must still be a valid configuration
        return vv * 2

    dfa_pkg.dfa_forward = fake_forward
    cfg = dfa_pkg.AttentionConfig(1000, 300, 2, 1, 4, [0])
    v = torch.arange(1000, dtype=torch.float32).view(1, 1000, 1, 1).expand(1, 1000, 1, 4).contiguous()
    out = ddist.segment_parallel_forward(v, v, v, dataclasses.replace(cfg))
    q.put((rank, out[0, :, 0, 0].tolist()))
    dist.destroy_process_group()


def test_segment_parallel_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_seg_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, rows in res:
        assert rows == [2.0 * i for i in range(1000)]


def _tail_worker(rank, world, port, q):
    """A shard holding only a tail segment shorter than w (N = 1000, w = 300,
    world 4: the last rank owns rows 900-999) and one shorter than r (N = 601,
    w = 300, r = 4: the last rank owns row 600 only)."""
    import dataclasses

    import paper_2403_09195_b200 as dfa_pkg
    from paper_2403_09195_b200 import dist as ddist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def fake_forward(qq, kk, vv, cfg, out=None, stream=None):
        cfg.validate()
        assert cfg.segment_len <= cfg.seq_len
        return vv * 2

    dfa_pkg.dfa_forward = fake_forward
    res = []
    for n, w, r in ((1000, 300, 2), (601, 300, 4)):
        cfg = dfa_pkg.AttentionConfig(n, w, r, 2, 4, [0, 1])
        v = torch.arange(n, dtype=torch.float32).view(1, n, 1, 1).expand(1, n, 2, 4).contiguous()
        out = ddist.segment_parallel_forward(v, v, v, dataclasses.replace(cfg))
        res.append(out[0, :, :, 0].tolist())
    q.put((rank, res))
    dist.destroy_process_group()


def test_segment_parallel_tail_shards_world4_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tail_worker, args=(r, 4, port, q)) for r in range(4)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(4)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, (a, b) in res:
        assert a == [[2.0 * i, 2.0 * i] for i in range(1000)]
        # rows 0-599: the stand-in kernel; row 600 (tail shorter than r = 4):
        # head 0 (gamma 0) keeps v's row, head 1 (gamma 1 >= 1 row) is 0
        assert b[:600] == [[2.0 * i, 2.0 * i] for i in range(600)]
        assert b[600] == [600.0, 0.0]
