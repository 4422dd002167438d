#!/usr/bin/env python3
"""Benchmark of the Dilated Flash Attention forward (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One "step" = one dfa_forward over one batch: BASELINE config 2 = 64 synthetic
1024x1024 images (N = 4096 tokens, 64x64 grid), h = 6 heads, d = 64,
(w, r) = (512, 2), head offsets j mod 2, bf16 in/out with fp32 accumulate.
`value` = images/s over all ranks (inputs resident in HBM); `tflops` counts
2 x flop_count().dilated_mults per image.  Multi-GPU: one process per GPU
(torchrun), every rank runs its own 64-image shard (weak scaling, no
collective on the hot path); after the timed steps the shards' outputs are
gathered to rank 0 over NCCL once and that gather is reported separately.

--impl reference times the reference's own CPU implementation
(oracle/_ref = the unmodified attnkit headers, or the C port if that .so is
absent) on the host cores, same workload definition, each step a bounded
sample of whole images.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_TOK, W, R, H, D = 4096, 512, 2, 6, 64
OFFSETS = [j % R for j in range(H)]
METRIC = "dilated-flash-attn TFLOP/s and images/s at 1024² (1/2/4/8 B200) vs CPU ref"
# Algorithmic work per (image, head): F = 2 * dilated_mults = 4*d*N*w/r^2;
# B = bf16 I/O: each kept q/k/v row read once + the full [N, d] output written.
FLOP_PER_UNIT = 4 * D * N_TOK * W // (R * R)
BYTES_PER_UNIT = 2 * D * N_TOK * 3 // R + 2 * D * N_TOK


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], "measured (MEASURED_PEAKS.json)"
    except (OSError, KeyError, ValueError):
        return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clock, power and clock-event (throttle) reasons sampled DURING the
    timed region through NVML (~every 0.5 ms, so even a few-ms region gets
    dozens of samples); nvidia-smi at 100 ms is the fallback
    (B200_PROFILING.md clocks line)."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, torch_device):
        self.dev = torch_device
        self.samples = []
        self.stop_flag = False
        self.thread = None
        self.nvml = None
        try:
            import pynvml as nv

            nv.nvmlInit()
            import torch

            pr = torch.cuda.get_device_properties(torch_device)
            bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0".encode()
            self.h = nv.nvmlDeviceGetHandleByPciBusId(bus)
            self.bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                         "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                         "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                         "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.nvml = nv
        except Exception:  # noqa: BLE001 -- no NVML: fall back to nvidia-smi
            self.nvml = None

    def _poll(self):
        nv = self.nvml
        n, watts = 0, 0.0
        while not self.stop_flag:
            try:
                if n % 16 == 0:  # power reads are the slow NVML query
                    watts = nv.nvmlDeviceGetPowerUsage(self.h) / 1e3
                self.samples.append((time.time(), nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM), watts,
                                     nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
                n += 1
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.0002)

    def start(self):
        if self.nvml:
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()

    def stop(self, t0, t1):
        if not self.nvml:
            return self._smi_once()
        self.stop_flag = True
        self.thread.join(timeout=2)
        window = [x for x in self.samples if t0 <= x[0] <= t1] or self.samples[-3:]
        if not window:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["no samples"]}
        reasons = sorted({n for x in window for n, bit in self.bits.items() if x[3] & bit})
        return {"sm_mhz": statistics.median(x[1] for x in window), "sm_max_mhz": self.max_mhz,
                "power_w_max": max(x[2] for x in window), "samples": len(window), "reasons": reasons,
                "sampler": "nvml ~0.5 ms during the timed region"}

    def _smi_once(self):
        try:
            out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw",
                                  "--format=csv,noheader,nounits", "-i", str(self.dev.index or 0)],
                                 capture_output=True, text=True, timeout=10).stdout.split(",")
            return {"sm_mhz": float(out[0]), "sm_max_mhz": float(out[1]), "power_w_max": float(out[2]),
                    "samples": 1, "reasons": [], "sampler": "nvidia-smi once (NVML unavailable)"}
        except Exception:  # noqa: BLE001
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}


def traffic_from_profiles(workload: str):
    """dram bytes per launch from the committed ncu --set full summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(workload)
    except (OSError, ValueError):
        return None


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_reference_images_per_s(target_s: float = 12.0, threads: int | None = None):
    """Time the reference CPU path on the host: (image, head) units of
    dilated_attention<float> at the config-2 geometry, one unit per thread at a
    time, all host threads.  Returns (images/s, cores, kind, sample)."""
    from oracle.oracle import Port, Reference, reference_available  # checker/baseline only

    threads = threads or cpu_threads()
    if reference_available():
        ref = Reference()
        probe = ref.time_dilated_f32(N_TOK, W, R, D, threads, threads, 8, 901)  # ~1 unit per thread
        units = max(threads, int(target_s / max(probe, 1e-3) * threads))
        units = ((units + H - 1) // H) * H
        secs = ref.time_dilated_f32(N_TOK, W, R, D, units, threads, 8, 902)
        kind = "reference"
    else:
        import numpy as np

        port = Port()
        rng = np.random.default_rng(901)
        q, k, v = (rng.standard_normal((4, N_TOK, D)).astype(np.float32) for _ in range(3))
        probe = port.time_dilated_f32(q, k, v, W, R, 1)
        units = max(H, int(target_s / max(probe, 1e-3)) // H * H)
        secs = port.time_dilated_f32(q, k, v, W, R, units)
        threads = 1
        kind = "port"
    imgs = units / H / secs
    sample = (f"{units} (image, head) units of dilated_attention<float> N={N_TOK} w={W} r={R} d={D}, "
              f"{threads} threads, {secs:.1f} s; images/s = units/{H}/s")
    return imgs, threads, kind, sample


# ------------------------------------------------------------ reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle.oracle import Port, Reference, reference_available

    threads = cpu_threads()
    # each step: ~8 units per host thread (so the thread pool stays busy
    # through the step), rounded up to whole images
    units = ((8 * threads + H - 1) // H) * H
    if reference_available():
        ref = Reference()
        kind = "reference"
        step = lambda s: ref.time_dilated_f32(N_TOK, W, R, D, units, threads, 8, 1000 + s)  # noqa: E731
    else:
        import numpy as np

        port = Port()
        kind = "port"
        threads = 1
        units = H
        rng = np.random.default_rng(901)
        q, k, v = (rng.standard_normal((2, N_TOK, D)).astype(np.float32) for _ in range(3))
        step = lambda s: port.time_dilated_f32(q, k, v, W, R, units)  # noqa: E731
    for s in range(args.warmup):
        step(s)
    times = [step(100 + s) for s in range(args.steps)]
    total = sum(times)
    imgs = units / H * args.steps / total
    tflops = FLOP_PER_UNIT * units * args.steps / total / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": imgs, "unit": "images/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(args, per_rank_batch=args.batch),
        "tflops": tflops,
        "cpu_baseline": {"value": imgs, "unit": "images/s", "cores": threads, "kind": kind,
                         "sample": f"per step {units} (image, head) units of the reference dilated_attention<float> "
                                   f"(N={N_TOK}, w={W}, r={R}, d={D}) over {threads} host threads"},
        "e2e": {"value": imgs, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(args, per_rank_batch):
    return {
        "workload": "config2: one SAM-Lightening attention layer, multi-head, 1024x1024 images "
                    "(N=4096 tokens, 64x64 grid), h=6, d=64, (w,r)=(512,2), offsets j mod 2, bf16 in/out",
        "batch_per_gpu": per_rank_batch, "global_batch": per_rank_batch * args.gpus, "seq_len": N_TOK,
        "heads": H, "head_dim": D, "segment_len": W, "interval": R, "head_offsets": OFFSETS,
        "parallelism": f"batch-shard x{args.gpus} (no hot-path collective)",
        "l2": "inputs+outputs 805 MB/step > 126 MB L2 (no flush needed)",
    }


# ----------------------------------------------------------------- B200 arm
def run_b200(args):
    import torch
    import torch.distributed as dist

    import paper_2403_09195_b200 as dfa

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    B = args.batch
    cfg = dfa.AttentionConfig(N_TOK, W, R, H, D, OFFSETS)
    assert dfa.query_path(cfg, "bf16", B) == 1, "tcgen05 path not selected for the bench workload"
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    q, k, v = (torch.randn((B, N_TOK, H, D), generator=g, device=dev, dtype=torch.bfloat16) for _ in range(3))
    o = torch.empty_like(q)
    stream = torch.cuda.current_stream(dev)

    def step():
        dfa.dfa_forward(q, k, v, cfg, out=o, stream=stream)

    sampler = ClockSampler(dev)
    sampler.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # One event pair around the K steps: the steps run back to back as they
    # would in a pipeline (programmatic dependent launch overlaps each
    # kernel's setup with the previous one's tail; an event record between
    # steps would serialise them).  Each step is one launch of the kernel, so
    # the kernel's average launch duration is the region / launches.
    e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    t_wall0 = time.time()
    e_start.record(stream)
    for i in range(args.steps):
        step()
        launches += dfa.last_launch_count()
    e_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_wall1 = time.time()
    total_ms = e_start.elapsed_time(e_end)
    clocks = sampler.stop(t_wall0, t_wall1)

    # max over ranks of the device-timed region
    t = torch.tensor([total_ms, total_ms / max(launches, 1)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, kernel_ms = t.tolist()
    images = B * world * args.steps
    imgs_s = images / (total_ms / 1e3)
    tflops = FLOP_PER_UNIT * H * images / (total_ms / 1e3) / 1e12

    # ---- final gather of the shards to rank 0 (outside the hot path)
    gather = None
    if world > 1:
        from paper_2403_09195_b200.dist import gather_to_rank0

        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        gathered = gather_to_rank0(o, B * world)
        e1.record(stream)
        torch.cuda.synchronize()
        gt = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
        dist.all_reduce(gt, op=dist.ReduceOp.MAX)
        gbytes = o.numel() * o.element_size() * (world - 1)
        gather = {"ms": gt.item(), "bytes_to_rank0": gbytes, "GBps": gbytes / (gt.item() / 1e3) / 1e9,
                  "how": "grouped ncclSend/ncclRecv of each shard's output to rank 0 (paper_2403_09195_b200.dist)"}
        del gathered

    # ---- end-to-end through the C-ABI host entry point (pinned host buffers)
    e2e = run_e2e(args, dfa, cfg, q, k, v, o, stream, world, dist, dev) if not args.quick else None

    if rank == 0:
        emit(args, world, B, imgs_s, tflops, total_ms, kernel_ms, launches, clocks, gather, e2e)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_e2e(args, dfa, cfg, q, k, v, o, stream, world, dist, dev):
    import torch

    B = q.shape[0]
    hq, hk, hv = (x.cpu().pin_memory() for x in (q, k, v))
    ho = torch.empty_like(hq).pin_memory()
    ws = dfa.Workspace(dfa.Workspace.bytes_for(cfg, "bf16", B))
    for _ in range(2):
        dfa.dfa_forward_host(hq, hk, hv, ho, cfg, ws, stream=stream)
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_steps = max(3, min(args.steps, 20))
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(e2e_steps):
        dfa.dfa_forward_host(hq, hk, hv, ho, cfg, ws, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    et = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    h2d, d2h = dfa.host_transfer_bytes(hq, hk, hv, cfg, "bf16")
    e2e = {"value": B * world * e2e_steps / (et.item() / 1e3), "unit": "images/s",
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "how": ("dfa_forward_host on pinned host buffers, per step: the tcgen05 kernel TMA-reads the kept q/k/v "
                   "rows straight from host memory over PCIe (zero-copy; h2d = those bytes), o comes back by "
                   "chunked D2H copies" if h2d < 3 * q.numel() * 2 else
                   "dfa_forward_host: H2D q,k,v from pinned memory + kernel + D2H o, per step")}
    ws.close()
    return e2e


def emit(args, world, B, imgs_s, tflops, total_ms, kernel_ms, launches, clocks, gather, e2e):
    if True:
        hbm_peak, tc_peak, src = peaks()
        bytes_launch = BYTES_PER_UNIT * H * B
        achieved = bytes_launch / (kernel_ms / 1e3) / 1e9
        workload_key = "config2_B64_h6_w512_r2"
        traffic = traffic_from_profiles(workload_key)
        line = {
            "metric": METRIC, "value": imgs_s, "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (torch.randn bf16, per-rank seed)",
            "config": workload_config(args, B),
            "tflops": tflops, "tensor_peak_frac": tflops / tc_peak,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": traffic,
                         "kernel": "dfa_sm100_kernel", "kernel_ms": kernel_ms,
                         "algorithmic_bytes_per_launch": bytes_launch, "peak_source": src,
                         "attainable_tflops": min(tc_peak, FLOP_PER_UNIT / BYTES_PER_UNIT * hbm_peak / 1e3)},
            "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
        }
        if gather:
            line["gather"] = gather
        if world == 1 and not args.no_cpu_baseline and not args.quick:
            imgs, cores, kind, sample = cpu_reference_images_per_s()
            line["cpu_baseline"] = {"value": imgs, "unit": "images/s", "cores": cores, "kind": kind,
                                    "sample": sample}
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="profiling mode: no e2e, no CPU baseline")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
