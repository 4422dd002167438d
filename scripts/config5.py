#!/usr/bin/env python3
"""BASELINE config 5: batch-sharded encoder attention over G GPUs -- 8192
synthetic 1024x1024 images (N = 4096 tokens), the 6 attention layers of the
SAM-Lightening encoder (h = 6, d = 64, (512, 2)), each rank running its
contiguous shard with no collective on the hot path, then ONE NCCL gather of
a per-image checksum of the final layer's output to rank 0 (the full outputs,
8192 x 3 MiB, stay sharded; `--gather-full` gathers a 64-image sample too).

    python scripts/config5.py                                   # 1 GPU
    torchrun --nproc-per-node G --master-addr 127.0.0.1 scripts/config5.py

Time = max over ranks of the device-timed sweep (CUDA events), images/s over
all ranks.  Layers use fresh synthetic q/k/v per (chunk, layer), generated
outside the timed region; chunks of --chunk images keep memory bounded.
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2403_09195_b200 as dfa  # noqa: E402
from paper_2403_09195_b200.dist import gather_to_rank0, shard_range  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--images", type=int, default=8192)
    ap.add_argument("--chunk", type=int, default=256)
    ap.add_argument("--layers", type=int, default=6)
    ap.add_argument("--gather-full", action="store_true")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    N, h, d = 4096, 6, 64
    cfg = dfa.AttentionConfig(N, 512, 2, h, d, dfa.AttentionConfig.spread_offsets(h, 2))
    lo, hi = shard_range(a.images, rank, world)
    mine = hi - lo
    C = min(a.chunk, mine)
    g = torch.Generator(device=dev).manual_seed(100 + rank)
    # one resident set of per-layer inputs for a chunk, reused across chunks
    # (synthetic data; the kernel cost does not depend on the values)
    layers = [[torch.randn((C, N, h, d), device=dev, dtype=torch.bfloat16, generator=g) for _ in range(3)]
              for _ in range(a.layers)]
    out = torch.empty_like(layers[0][0])
    sums = torch.zeros(mine, device=dev, dtype=torch.float32)

    def sweep():
        for c0 in range(0, mine, C):
            n = min(C, mine - c0)
            for (q, k, v) in layers:
                dfa.dfa_forward(q[:n], k[:n], v[:n], cfg, out=out[:n])
            sums[c0:c0 + n] = out[:n].float().sum(dim=(1, 2, 3))

    sweep()  # warm
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sweep()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = t.item()
    res = {"config": "config5: 8192 images x 6 encoder attention layers (h=6, d=64, (512,2)), batch-sharded",
           "n_gpus": world, "images": a.images, "ms": ms, "images_per_s": a.images / (ms / 1e3),
           "tflops": 2 * dfa.flop_count(cfg).dilated_mults * a.images * a.layers / (ms / 1e3) / 1e12}
    if world > 1:
        e0.record()
        allsums = gather_to_rank0(sums, a.images)
        e1.record()
        torch.cuda.synchronize()
        res["gather_checksums_ms"] = e0.elapsed_time(e1)
        if a.gather_full:
            sample = out[: max(1, 64 // world)].contiguous()
            full = gather_to_rank0(sample, sample.shape[0] * world)
            del full
    else:
        allsums = sums
    if rank == 0:
        res["checksum_of_checksums"] = float(allsums.double().sum().item())
        print(json.dumps(res))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
