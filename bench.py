#!/usr/bin/env python3
"""Benchmark of the Dilated Flash Attention forward (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload config2|config1|config3|config4|lse|config5]

Workloads (BASELINE.json configs; N = 4096 tokens = the 64x64 grid of a
1024x1024 image, d = 64, synthetic N(0, 1) inputs):
  config2 (default)  one SAM-Lightening attention layer, B = 64 images per GPU,
                     h = 6, (w, r) = (512, 2), offsets j mod 2, bf16 in/out with
                     fp32 accumulate.  One step = one dfa_forward over the batch.
  config1            fp32 validation mode, B = 1, h = 1, (512, 2), offset 0.
  config3            the 6 attention layers of the encoder (fresh q/k/v each),
                     h = 6, (512, 2), batch --batch (sweep 1..256 in the default
                     run's extras); one step = 6 launches from a CUDA graph.
  config4            the (w, r) grid w in {256..4096} x r in {1,2,4,8}, B = 64,
                     h = 6; one step = all 20 branch launches.
  lse                LSE-combined LongNet set {(512,1),(1024,2),(2048,4),(4096,8)}
                     (extension), B = 64, h = 6; one step = one multibranch call.
  config5            8192 images x 6 layers, batch-sharded over the ranks (strong
                     scaling), then one NCCL gather of the outputs to rank 0
                     (reported separately, outside the timed region).

`value` = images/s over all ranks (inputs resident in HBM); `tflops` counts
2 x flop_count().dilated_mults per (image, head, layer).  The default run
(N = 1, config2) also times configs 1, 3, 4 and the LSE set and puts them,
each with its own NVML clock record, under `extras`.

Multi-GPU: one process per GPU.  Under torchrun (WORLD_SIZE set) every rank
runs its shard; a plain `python bench.py --gpus N` re-launches itself under
torch.distributed.run with N ranks (and fails if fewer than N GPUs are
visible).  The timed region is bracketed by barrier + synchronize on both
sides and the max over ranks is reported; there is no collective on the
hot path.

--impl reference times the reference's own CPU implementation
(oracle/_ref = the unmodified attnkit headers compiled here, or the C port
if that .so is absent) on the host cores, same workload definition, each
step a bounded sample of whole images.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_TOK, D = 4096, 64
W, R, H = 512, 2, 6  # the headline geometry (configs 1-3, 5)
LAYERS = 6
METRIC = "dilated-flash-attn TFLOP/s and images/s at 1024² (1/2/4/8 B200) vs CPU ref"
GRID_W = (256, 512, 1024, 2048, 4096)
GRID_R = (1, 2, 4, 8)
LSE_SET = [(512, 1), (1024, 2), (2048, 4), (4096, 8)]
CONFIG5_IMAGES = 8192
L2_BYTES = 126 * 2 ** 20
WORKLOADS = ("config2", "config1", "config3", "config4", "lse", "config5")


def flop_per_unit(w, r, d=D, n=N_TOK):
    """2 x dilated_mults of one (image, head) at exact division: 4 d N w / r^2."""
    return 4 * d * n * w // (r * r)


def bytes_per_unit(r, es=2, d=D, n=N_TOK):
    """Each kept q/k/v row read once + the full [N, d] output written (zero rows too)."""
    return es * d * (n // r) * 3 + es * d * n


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], "measured (MEASURED_PEAKS.json)"
    except (OSError, KeyError, ValueError):
        return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clock, power and clock-event (throttle) reasons sampled DURING a
    timed region through NVML (~every 0.5 ms, so even a few-ms region gets
    dozens of samples); nvidia-smi at 100 ms is the fallback
    (B200_PROFILING.md clocks line)."""

    def __init__(self, torch_device):
        self.dev = torch_device
        self.samples = []
        self.stop_flag = False
        self.thread = None
        self.nvml = None
        try:
            import pynvml as nv
            import torch

            nv.nvmlInit()
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
        """Poll from now until close(); window() reads any timed region."""
        if self.nvml and self.thread is None:
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            time.sleep(0.02)  # first samples land before the first region

    def close(self):
        self.stop_flag = True
        if self.thread is not None:
            self.thread.join(timeout=2)

    def window(self, t0, t1):
        if not self.nvml:
            return self._smi_once()
        samples = list(self.samples)
        win = [x for x in samples if t0 <= x[0] <= t1]
        if not win:  # region shorter than one NVML poll: the samples bracketing it
            before = [x for x in samples if x[0] < t0][-1:]
            after = [x for x in samples if x[0] > t1][:1]
            win = before + after
        if not win:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["no samples"]}
        reasons = sorted({n for x in win for n, bit in self.bits.items() if x[3] & bit})
        return {"sm_mhz": statistics.median(x[1] for x in win), "sm_max_mhz": self.max_mhz,
                "power_w_max": max(x[2] for x in win), "samples": len(win), "reasons": reasons,
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


def host_info():
    """CPU model (lscpu / /proc/cpuinfo) and the compiler that built the reference checker."""
    model = platform.processor() or "unknown"
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:  # noqa: BLE001
        try:
            with open("/proc/cpuinfo") as f:
                for line in f:
                    if line.startswith("model name"):
                        model = line.split(":", 1)[1].strip()
                        break
        except OSError:
            pass
    compiler = None
    info = os.path.join(ROOT, "oracle", "_ref", "BUILD_INFO")
    try:
        with open(info) as f:
            compiler = f.read().strip()
    except OSError:
        try:
            compiler = subprocess.run(["g++", "--version"], capture_output=True, text=True,
                                      timeout=10).stdout.splitlines()[0] + " (-O3 -ffp-contract=off)"
        except Exception:  # noqa: BLE001
            compiler = None
    return {"cpu_model": model, "nproc": os.cpu_count(), "threads_used": cpu_threads(), "compiler": compiler}


def reference_geometry(workload):
    """(w, r, units per image) of the reference arm's unit for a workload."""
    if workload == "config1":
        return W, R, 1
    if workload in ("config3", "config5"):
        return W, R, H * LAYERS
    return W, R, H


def cpu_reference_images_per_s(workload="config2", target_s: float = 12.0, threads: int | None = None):
    """Time the reference CPU path on the host: (image, head) units of
    dilated_attention<float> at the workload's geometry, one unit per thread at
    a time, all host threads.  Returns (images/s, cores, kind, sample)."""
    from oracle.oracle import Port, Reference, reference_available  # checker/baseline only

    w, r, per_img = reference_geometry(workload)
    threads = threads or cpu_threads()
    if reference_available():
        ref = Reference()
        probe = ref.time_dilated_f32(N_TOK, w, r, D, threads, threads, 8, 901)  # ~1 unit per thread
        units = max(threads, int(target_s / max(probe, 1e-3) * threads))
        units = ((units + per_img - 1) // per_img) * per_img
        secs = ref.time_dilated_f32(N_TOK, w, r, D, units, threads, 8, 902)
        kind = "reference"
    else:
        import numpy as np

        port = Port()
        rng = np.random.default_rng(901)
        q, k, v = (rng.standard_normal((4, N_TOK, D)).astype(np.float32) for _ in range(3))
        probe = port.time_dilated_f32(q, k, v, w, r, 1)
        units = max(per_img, int(target_s / max(probe, 1e-3)) // per_img * per_img)
        secs = port.time_dilated_f32(q, k, v, w, r, units)
        threads = 1
        kind = "port"
    imgs = units / per_img / secs
    sample = (f"{units} (image, head[, layer]) units of dilated_attention<float> N={N_TOK} w={w} r={r} d={D}, "
              f"{threads} threads, {secs:.1f} s; images/s = units/{per_img}/s")
    return imgs, threads, kind, sample


# ------------------------------------------------------------ reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle.oracle import Port, Reference, reference_available

    w, r, per_img = reference_geometry(args.workload)
    threads = cpu_threads()
    # each step: ~8 units per host thread (so the thread pool stays busy
    # through the step), rounded up to whole images
    units = ((8 * threads + per_img - 1) // per_img) * per_img
    if reference_available():
        ref = Reference()
        kind = "reference"
        step = lambda s: ref.time_dilated_f32(N_TOK, w, r, D, units, threads, 8, 1000 + s)  # noqa: E731
    else:
        import numpy as np

        port = Port()
        kind = "port"
        threads = 1
        units = per_img
        rng = np.random.default_rng(901)
        q, k, v = (rng.standard_normal((2, N_TOK, D)).astype(np.float32) for _ in range(3))
        step = lambda s: port.time_dilated_f32(q, k, v, w, r, units)  # noqa: E731
    for s in range(args.warmup):
        step(s)
    times = [step(100 + s) for s in range(args.steps)]
    total = sum(times)
    imgs = units / per_img * args.steps / total
    tflops = flop_per_unit(w, r) * units * args.steps / total / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": imgs, "unit": "images/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "strong" if args.workload == "config5" else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(args.workload, args, args.batch),
        "tflops": tflops,
        "cpu_baseline": {"value": imgs, "unit": "images/s", "cores": threads, "kind": kind,
                         "sample": f"per step {units} (image, head[, layer]) units of the reference "
                                   f"dilated_attention<float> (N={N_TOK}, w={w}, r={r}, d={D}) over {threads} "
                                   f"host threads", **host_info()},
        "e2e": {"value": imgs, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(name, args, batch):
    world = args.gpus
    common = {"seq_len": N_TOK, "head_dim": D, "grid": "64x64 tokens of a 1024x1024 image"}
    if name == "config1":
        return {"workload": "config1: single-head dilated_attention<float>, B=1, N=4096, (w,r)=(512,2), offset 0, "
                            "fp32 validation mode (SIMT kernel)", "batch_per_gpu": 1, "global_batch": world,
                "heads": 1, "segment_len": W, "interval": R, **common,
                "parallelism": f"replicas x{world}",
                "l2": "64 rotating input sets (256 MB > 126 MB L2)"}
    if name == "config3":
        return {"workload": f"config3: the 6 encoder attention layers (fresh q/k/v per layer), h=6, (w,r)=(512,2), "
                            f"bf16, CUDA graph of 6 launches", "batch_per_gpu": batch, "global_batch": batch * world,
                "heads": H, "layers": LAYERS, "segment_len": W, "interval": R, **common,
                "parallelism": f"batch-shard x{world}",
                "l2": "rotating layer sets so every step's inputs exceed 2x the 126 MB L2"}
    if name == "config4":
        return {"workload": "config4: (w,r) grid w in {256,512,1024,2048,4096} x r in {1,2,4,8}, B=64, h=6, "
                            "offsets j mod r, bf16; one step = the 20 branch launches",
                "batch_per_gpu": 64, "global_batch": 64 * world, "heads": H, **common,
                "parallelism": f"batch-shard x{world}", "l2": "inputs+outputs 805 MB > L2"}
    if name == "lse":
        return {"workload": "lse: LSE-combined branch set {(512,1),(1024,2),(2048,4),(4096,8)} (extension), "
                            "B=64, h=6, offsets j mod r, bf16", "batch_per_gpu": 64, "global_batch": 64 * world,
                "heads": H, "branches": LSE_SET, **common, "parallelism": f"batch-shard x{world}",
                "l2": "inputs+outputs 805 MB > L2"}
    if name == "config5":
        return {"workload": f"config5: {CONFIG5_IMAGES} images x 6 encoder attention layers, h=6, (w,r)=(512,2), "
                            f"bf16, batch-sharded over {world} GPU(s), final NCCL gather outside the timed region",
                "global_batch": CONFIG5_IMAGES, "heads": H, "layers": LAYERS, "segment_len": W, "interval": R,
                **common, "parallelism": f"batch-shard x{world} (no hot-path collective)",
                "l2": "per-layer inputs >= 3 GB > L2", "data_note": "layers share one synthetic q/k/v set"}
    return {"workload": "config2: one SAM-Lightening attention layer, multi-head, 1024x1024 images "
                        "(N=4096 tokens, 64x64 grid), h=6, d=64, (w,r)=(512,2), offsets j mod 2, bf16 in/out",
            "batch_per_gpu": batch, "global_batch": batch * world, "seq_len": N_TOK,
            "heads": H, "head_dim": D, "segment_len": W, "interval": R, "head_offsets": [j % R for j in range(H)],
            "parallelism": f"batch-shard x{world} (no hot-path collective)",
            "l2": "inputs+outputs 805 MB/step > 126 MB L2 (no flush needed)"}


# ----------------------------------------------------------------- B200 arm
class Ctx:
    """Per-rank state shared by the workloads."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist

        import paper_2403_09195_b200 as dfa

        self.torch, self.dist, self.dfa, self.args = torch, dist, dfa, args
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        if self.world > 1:
            dist.init_process_group("nccl", device_id=self.dev)
        self.stream = torch.cuda.current_stream(self.dev)
        self.sampler = ClockSampler(self.dev)
        self.sampler.start()

    def cfg(self, w, r, h=H, d=D, n=N_TOK):
        return self.dfa.AttentionConfig(n, w, r, h, d, self.dfa.AttentionConfig.spread_offsets(h, r))

    def randn(self, shape, seed, dtype=None):
        torch = self.torch
        g = torch.Generator(device=self.dev).manual_seed(seed + 7919 * self.rank)
        return torch.randn(shape, generator=g, device=self.dev, dtype=dtype or torch.bfloat16)

    def barrier(self):
        self.torch.cuda.synchronize()
        if self.world > 1:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def max_over_ranks(self, *vals):
        t = self.torch.tensor(list(vals), device=self.dev, dtype=self.torch.float64)
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return t.tolist()

    def timed(self, step, steps, warmup):
        """W warm-up steps, then K steps back to back between one CUDA-event pair
        on the launching stream, barrier + synchronize on both sides; clocks
        sampled during the region.  Returns (total_ms max over ranks, launches, clocks)."""
        torch = self.torch
        for _ in range(warmup):
            step()
        self.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        launches = 0
        t0 = time.time()
        e0.record(self.stream)
        for _ in range(steps):
            launches += step() or 0
        e1.record(self.stream)
        self.barrier()
        t1 = time.time()
        clocks = self.sampler.window(t0, t1)
        total_ms, = self.max_over_ranks(e0.elapsed_time(e1))
        return total_ms, launches, clocks


def roofline_line(kernel_ms, bytes_launch, flop_launch, kernel, workload_key):
    hbm_peak, tc_peak, src = peaks()
    achieved = bytes_launch / (kernel_ms / 1e3) / 1e9
    ai = flop_launch / bytes_launch
    bound = "tensor" if ai * hbm_peak / 1e3 >= tc_peak else "hbm"
    tf = flop_launch / (kernel_ms / 1e3) / 1e12
    if bound == "tensor":
        return {"bound": "tensor", "achieved": tf, "peak": tc_peak, "unit": "TFLOP/s", "frac": tf / tc_peak,
                "traffic": traffic_from_profiles(workload_key), "kernel": kernel, "kernel_ms": kernel_ms,
                "algorithmic_flop_per_launch": flop_launch, "algorithmic_bytes_per_launch": bytes_launch,
                "hbm_GBps": achieved, "peak_source": src}
    return {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
            "traffic": traffic_from_profiles(workload_key), "kernel": kernel, "kernel_ms": kernel_ms,
            "algorithmic_bytes_per_launch": bytes_launch, "peak_source": src,
            "attainable_tflops": min(tc_peak, ai * hbm_peak / 1e3), "tflops": tf}


def wl_config2(ctx, steps, warmup, batch, with_e2e=True):
    dfa = ctx.dfa
    cfg = ctx.cfg(W, R)
    assert dfa.query_path(cfg, "bf16", batch) == 1, "tcgen05 path not selected for the bench workload"
    q, k, v = (ctx.randn((batch, N_TOK, H, D), 1234 + i) for i in range(3))
    o = ctx.torch.empty_like(q)

    def step():
        dfa.dfa_forward(q, k, v, cfg, out=o, stream=ctx.stream)
        return dfa.last_launch_count()

    # Steps run back to back between one event pair (programmatic dependent
    # launch overlaps each kernel's setup with the previous one's tail; an
    # event record between steps would serialise them).  One launch per step,
    # so the kernel's average launch duration is region / launches.
    total_ms, launches, clocks = ctx.timed(step, steps, warmup)
    images = batch * ctx.world * steps
    _, tc_peak, _ = peaks()
    tf = flop_per_unit(W, R) * H * images / (total_ms / 1e3) / 1e12
    kernel_ms = total_ms / launches if launches else total_ms / steps
    res = {"value": images / (total_ms / 1e3), "unit": "images/s", "ms_per_step": total_ms / steps,
           "tflops": tf, "tensor_peak_frac": tf / tc_peak, "gpu_launches": launches, "clocks": clocks,
           "roofline": roofline_line(kernel_ms, bytes_per_unit(R) * H * batch, flop_per_unit(W, R) * H * batch,
                                     "dfa_sm100_kernel", "config2_B64_h6_w512_r2"),
           "scaling": "weak", "dtype": "bf16"}
    if with_e2e:
        res["e2e"] = e2e_config2(ctx, cfg, q, k, v, steps)
    res["_out"] = o
    return res


def e2e_config2(ctx, cfg, q, k, v, steps):
    """The same metric through the C-ABI host entry point dfa_forward_host on
    pinned host buffers: every step moves that step's inputs host -> device
    and the output back, inside the timed region."""
    torch, dfa = ctx.torch, ctx.dfa
    B = q.shape[0]
    hq, hk, hv = (x.cpu().pin_memory() for x in (q, k, v))
    ho = torch.empty_like(hq).pin_memory()
    ws = dfa.Workspace(dfa.Workspace.bytes_for(cfg, "bf16", B))
    for _ in range(2):
        dfa.dfa_forward_host(hq, hk, hv, ho, cfg, ws, stream=ctx.stream)
    ctx.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = max(3, min(steps, 20))
    e0.record(ctx.stream)
    for _ in range(n):
        dfa.dfa_forward_host(hq, hk, hv, ho, cfg, ws, stream=ctx.stream)
    e1.record(ctx.stream)
    ctx.barrier()
    et, = ctx.max_over_ranks(e0.elapsed_time(e1))
    h2d, d2h = dfa.host_transfer_bytes(hq, hk, hv, cfg, "bf16", out=ho)
    ws.close()
    return {"value": B * ctx.world * n / (et / 1e3), "unit": "images/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": n,
            "how": ("dfa_forward_host on pinned host buffers, per step: the tcgen05 kernel TMA-reads the kept q/k/v "
                    "rows straight from host memory over PCIe and TMA-writes the kept o rows straight into the "
                    "host output (zero-copy both ways; h2d / d2h = those bytes), while host threads zero-fill "
                    "the o rows no view keeps" if d2h < q.numel() * 2 else
                    "dfa_forward_host on pinned host buffers, per step: the tcgen05 kernel TMA-reads the kept q/k/v "
                    "rows straight from host memory over PCIe (zero-copy; h2d = those bytes), o comes back by "
                    "chunked D2H copies" if h2d < 3 * q.numel() * 2 else
                    "dfa_forward_host: H2D q,k,v from pinned memory + kernel + D2H o, per step")}


def wl_config1(ctx, steps, warmup):
    """fp32 single head, B = 1: a latency workload.  64 rotating input sets
    (256 MB > L2), the calls replayed from a CUDA graph so the device time of
    the kernels -- not the Python launch path -- is measured."""
    torch, dfa = ctx.torch, ctx.dfa
    cfg = dfa.AttentionConfig(N_TOK, W, R, 1, D, [0])
    n_sets = 64
    sets = [[ctx.randn((1, N_TOK, 1, D), 50 + 3 * s + i, torch.float32) for i in range(3)] for s in range(n_sets)]
    outs = [torch.empty_like(sets[0][0]) for _ in range(n_sets)]
    for (q, k, v), o in zip(sets, outs):
        dfa.dfa_forward(q, k, v, cfg, out=o)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream(ctx.dev)
    s.wait_stream(ctx.stream)
    launches = 0
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for (q, k, v), o in zip(sets, outs):
                dfa.dfa_forward(q, k, v, cfg, out=o, stream=s)
                launches += dfa.last_launch_count()
    ctx.stream.wait_stream(s)
    reps = max(1, steps // n_sets)

    def step():
        g.replay()
        return launches

    total_ms, total_launches, clocks = ctx.timed(step, reps, max(3, warmup // n_sets))
    calls = n_sets * reps
    ms = total_ms / calls
    _, tc_peak, _ = peaks()
    # e2e: the reference-shaped single-head host call (dfa_dilated_attention_host)
    hq, hk, hv = (x.view(N_TOK, D).cpu().pin_memory() for x in sets[0])
    ho = torch.empty_like(hq).pin_memory()
    ws = dfa.Workspace(dfa.Workspace.bytes_for(cfg, "f32", 1))
    for _ in range(3):
        dfa.dfa_forward_host(hq.view(1, N_TOK, 1, D), hk.view(1, N_TOK, 1, D), hv.view(1, N_TOK, 1, D),
                             ho.view(1, N_TOK, 1, D), cfg, ws, dtype="f32", stream=ctx.stream)
    ctx.barrier()
    n = 50
    t0 = time.perf_counter()
    for _ in range(n):
        dfa.dfa_forward_host(hq.view(1, N_TOK, 1, D), hk.view(1, N_TOK, 1, D), hv.view(1, N_TOK, 1, D),
                             ho.view(1, N_TOK, 1, D), cfg, ws, dtype="f32", stream=ctx.stream)
    e2e_s = (time.perf_counter() - t0) / n
    h2d, d2h = dfa.host_transfer_bytes(hq.view(1, N_TOK, 1, D), hk.view(1, N_TOK, 1, D), hv.view(1, N_TOK, 1, D),
                                       cfg, "f32", out=ho.view(1, N_TOK, 1, D))
    ws.close()
    return {"value": ctx.world / (ms / 1e3), "unit": "images/s", "ms_per_step": ms, "us_per_call": ms * 1e3,
            "tflops": flop_per_unit(W, R) / (ms / 1e3) / 1e12 * ctx.world, "gpu_launches": total_launches,
            "clocks": clocks, "dtype": "f32", "scaling": "weak", "timed_calls": calls,
            "e2e": {"value": ctx.world / e2e_s, "unit": "images/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "us_per_call": e2e_s * 1e6,
                    "how": "dfa_forward_host (synchronous host-buffer call, wall clock incl. H2D + kernel + D2H)"}}


def config3_step(ctx, batch):
    """CUDA graph of the 6 layer launches over rotating layer sets whose
    inputs exceed 2x the L2.  Returns (replay fn, sets per replay, launches per replay)."""
    torch, dfa = ctx.torch, ctx.dfa
    cfg = ctx.cfg(W, R)
    per_layer = 4 * batch * N_TOK * H * D * 2  # q, k, v, o
    n_sets = max(1, -(-2 * L2_BYTES // (per_layer * LAYERS)))
    sets = []
    for s in range(n_sets):
        layers = [[ctx.randn((batch, N_TOK, H, D), 300 + 17 * s + 3 * layer + i) for i in range(3)]
                  for layer in range(LAYERS)]
        sets.append((layers, [torch.empty_like(layers[0][0]) for _ in range(LAYERS)]))
    for layers, outs in sets:
        for (q, k, v), o in zip(layers, outs):
            dfa.dfa_forward(q, k, v, cfg, out=o)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream(ctx.dev)
    s.wait_stream(ctx.stream)
    launches = 0
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for layers, outs in sets:
                for (q, k, v), o in zip(layers, outs):
                    dfa.dfa_forward(q, k, v, cfg, out=o, stream=s)
                    launches += dfa.last_launch_count()
    ctx.stream.wait_stream(s)
    return g, n_sets, launches, sets


def wl_config3(ctx, steps, warmup, batch):
    g, n_sets, launches, keep = config3_step(ctx, batch)

    def step():
        g.replay()
        return launches

    reps = max(1, steps // n_sets)
    total_ms, total_launches, clocks = ctx.timed(step, reps, max(3, warmup // n_sets))
    ms = total_ms / (reps * n_sets)  # one step = the 6 layers of one batch
    _, tc_peak, _ = peaks()
    tf = flop_per_unit(W, R) * H * LAYERS * batch * ctx.world / (ms / 1e3) / 1e12
    del keep
    return {"value": batch * ctx.world / (ms / 1e3), "unit": "images/s", "ms_per_step": ms, "tflops": tf,
            "tensor_peak_frac": tf / tc_peak, "gpu_launches": total_launches, "clocks": clocks, "dtype": "bf16",
            "scaling": "weak", "batch": batch, "rotating_sets": n_sets}


def wl_config4(ctx, steps, warmup):
    """Every (w, r) of the grid: ms, TFLOP/s, algorithmic GB/s, fraction of the
    attainable min(peak, AI x HBM) -- each cell timed on its own (K launches
    back to back) with its own clock record; the workload's value is images/s
    through the whole grid (one step = the 20 launches)."""
    dfa = ctx.dfa
    hbm, tc, _ = peaks()
    B = 64
    q, k, v = (ctx.randn((B, N_TOK, H, D), 77 + i) for i in range(3))
    o = ctx.torch.empty_like(q)
    rows, total_ms, launches = [], 0.0, 0
    per_cell = max(5, steps // 2)
    for w in GRID_W:
        for r in GRID_R:
            cfg = ctx.cfg(w, r)

            def step(cfg=cfg):
                dfa.dfa_forward(q, k, v, cfg, out=o, stream=ctx.stream)
                return dfa.last_launch_count()

            t, n, clocks = ctx.timed(step, per_cell, warmup)
            ms = t / per_cell
            fl = flop_per_unit(w, r) * H * B
            by = bytes_per_unit(r) * H * B
            ai = fl / by
            attain = min(tc, ai * hbm / 1e3)
            tf = fl / (ms / 1e3) / 1e12
            rows.append({"w": w, "r": r, "ms": ms, "tflops": tf, "GBps": by / (ms / 1e3) / 1e9, "AI": ai,
                         "attainable_tflops": attain, "frac_of_attainable": tf / attain,
                         "frac_of_tensor_peak": tf / tc, "bound": "tensor" if ai * hbm / 1e3 >= tc else "hbm",
                         "path": "tcgen05" if dfa.query_path(cfg, "bf16", B) == 1 else "simt",
                         "sm_mhz": clocks.get("sm_mhz"), "reasons": clocks.get("reasons")})
            total_ms += ms
            launches += n
    return {"value": B * ctx.world / (total_ms / 1e3), "unit": "images/s (through the 20-branch grid)",
            "ms_per_step": total_ms, "gpu_launches": launches, "dtype": "bf16", "scaling": "weak", "rows": rows}


def wl_lse(ctx, steps, warmup):
    """LSE-combined LongNet set (extension, north_star item 3): the fused
    single-kernel path (every branch + the combine in one tcgen05 launch) and,
    timed beside it, the per-branch path (one launch per branch, epilogue merge)."""
    torch, dfa = ctx.torch, ctx.dfa
    from paper_2403_09195_b200 import _lib, multibranch_mode

    hbm, tc, _ = peaks()
    B = 64
    q, k, v = (ctx.randn((B, N_TOK, H, D), 91 + i) for i in range(3))
    o = torch.empty_like(q)
    cfg = ctx.cfg(512, 1)
    ws = torch.empty(1 << 28, dtype=torch.uint8, device=ctx.dev)

    def step():
        dfa.dfa_forward_multibranch(q, k, v, cfg, LSE_SET, out=o, workspace=ws, stream=ctx.stream)
        return dfa.last_launch_count()

    total_ms, launches, clocks = ctx.timed(step, steps, warmup)
    with multibranch_mode(_lib.DFA_MB_PER_BRANCH):
        pb_ms, pb_launches, pb_clocks = ctx.timed(step, steps, warmup)
    ms, pb = total_ms / steps, pb_ms / steps
    fl = sum(flop_per_unit(w, r) for w, r in LSE_SET) * H * B
    by = (3 * 2 * D * N_TOK + 2 * D * N_TOK) * H * B  # q, k, v read once + o written once (fused ideal)
    tf = fl / (ms / 1e3) / 1e12
    return {"value": B * ctx.world / (ms / 1e3), "unit": "images/s", "ms_per_step": ms, "tflops": tf,
            "tensor_peak_frac": tf / tc, "gpu_launches": launches, "clocks": clocks, "dtype": "bf16",
            "scaling": "weak", "branches": LSE_SET, "launches_per_call": launches // max(1, steps),
            "kernel": "dfa_mb_sm100_kernel (all branches + LSE combine, one launch)", "AI_fused": fl / by,
            "per_branch": {"ms_per_step": pb, "tflops": fl / (pb / 1e3) / 1e12,
                           "launches_per_call": pb_launches // max(1, steps), "clocks": pb_clocks}}


def wl_frows(ctx, steps, warmup):
    """SURVEY §8(f) rows at config-2 shapes (B = 64, N = 4096, h = 6, (512, 2),
    bf16), each timed back to back with its own clock record: the backward of
    the core (Delta pass + tcgen05 backward), the multi-head layer
    (multi_head_dilated: class-split QKV GEMM + core + Wo GEMM, own tcgen05
    GEMM) and one encoder block (LN, attention mix, LN, erf-GELU MLP)."""
    torch, dfa = ctx.torch, ctx.dfa
    hbm, tc, _ = peaks()
    B, Dm, hidden = 64, H * D, 4 * H * D
    cfg = ctx.cfg(W, R)
    fwd_flop = flop_per_unit(W, R) * H * B
    out = {}
    q, k, v, do = (ctx.randn((B, N_TOK, H, D), 131 + i) for i in range(4))
    L = torch.empty((B, H, N_TOK), device=ctx.dev, dtype=torch.float32)
    o = dfa.dfa_forward(q, k, v, cfg, lse=L, stream=ctx.stream)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    ws = torch.empty(B * H * N_TOK * 4 + 256, dtype=torch.uint8, device=ctx.dev)

    def bwd():
        dfa.dfa_backward(q, k, v, o, L, do, cfg, dq, dk, dv, workspace=ws, stream=ctx.stream)
        return dfa.last_launch_count()

    t, n, clk = ctx.timed(bwd, steps, warmup)
    ms = t / steps
    kept = B * H * (N_TOK // R) * D * 2
    by = 5 * kept + B * H * (N_TOK // R) * 4 * 2 + 3 * B * N_TOK * H * D * 2  # q,k,v,o,dO kept rows + lse, Delta + dq,dk,dv
    out["backward"] = {"ms": ms, "tflops": 2.5 * fwd_flop / (ms / 1e3) / 1e12, "GBps": by / (ms / 1e3) / 1e9,
                       "hbm_frac": by / (ms / 1e3) / 1e9 / hbm, "algorithmic_bytes": by,
                       "launches_per_call": n // max(1, steps), "clocks": clk}
    del q, k, v, do, o, dq, dk, dv, L, ws
    x = ctx.randn((B, N_TOK, Dm), 141)
    g = torch.Generator(device=ctx.dev).manual_seed(7)
    wq, wk, wv = (torch.randn((H, Dm, D), device=ctx.dev, dtype=torch.bfloat16, generator=g) / Dm ** 0.5
                  for _ in range(3))
    wo = torch.randn((Dm, Dm), device=ctx.dev, dtype=torch.bfloat16, generator=g) / Dm ** 0.5
    y = torch.empty_like(x)
    wsp = torch.empty(4 * B * N_TOK * Dm * 2 + (40 << 20), dtype=torch.uint8, device=ctx.dev)

    def mh():
        dfa.multi_head_dilated(x, wq, wk, wv, wo, cfg, out=y, workspace=wsp, stream=ctx.stream)
        return dfa.last_launch_count()

    t, n, clk = ctx.timed(mh, steps, warmup)
    ms = t / steps
    proj = 2 * B * N_TOK * Dm * Dm * 4 // R  # executed: the class split does 1/r of the dense projections
    out["multihead"] = {"ms": ms, "images_per_s": B / (ms / 1e3), "tflops": (proj + fwd_flop) / (ms / 1e3) / 1e12,
                        "launches_per_call": n // max(1, steps), "clocks": clk}
    s = 1.0 / Dm ** 0.5
    prm = {"ln1_g": torch.ones(Dm), "ln1_b": torch.zeros(Dm), "wq": s * torch.randn(H, Dm, D),
           "wk": s * torch.randn(H, Dm, D), "wv": s * torch.randn(H, Dm, D), "wo": s * torch.randn(Dm, Dm),
           "bo": torch.zeros(Dm), "ln2_g": torch.ones(Dm), "ln2_b": torch.zeros(Dm),
           "w1": s * torch.randn(Dm, hidden), "b1": torch.zeros(hidden), "w2": torch.randn(hidden, Dm) / hidden ** 0.5,
           "b2": torch.zeros(Dm)}
    prm = {kk: vv.to(ctx.dev, torch.bfloat16).contiguous() for kk, vv in prm.items()}
    wsb = torch.empty(7 * B * N_TOK * Dm * 2 + 2 * B * N_TOK * hidden * 2 + (40 << 20), dtype=torch.uint8,
                      device=ctx.dev)

    def blk():
        dfa.encoder_block_forward(x, prm, cfg, out=y, workspace=wsb, stream=ctx.stream)
        return dfa.last_launch_count()

    t, n, clk = ctx.timed(blk, max(3, steps // 2), warmup)
    ms = t / max(3, steps // 2)
    bf = proj + fwd_flop + 2 * 2 * B * N_TOK * Dm * hidden
    out["block"] = {"ms": ms, "images_per_s": B / (ms / 1e3), "tflops": bf / (ms / 1e3) / 1e12,
                    "launches_per_call": n // max(1, max(3, steps // 2)), "clocks": clk}
    return out


def wl_config5(ctx, steps, warmup):
    """8192 images x 6 layers, contiguous image shards per rank; the final NCCL
    gather of every image's output to rank 0 runs after the timed region and
    is reported under `gather`."""
    torch, dfa = ctx.torch, ctx.dfa
    from paper_2403_09195_b200.dist import gather_to_rank0, shard_range

    lo, hi = shard_range(CONFIG5_IMAGES, ctx.rank, ctx.world)
    mine = hi - lo
    cfg = ctx.cfg(W, R)
    q, k, v = (ctx.randn((mine, N_TOK, H, D), 500 + i) for i in range(3))
    o = torch.empty_like(q)

    def step():
        n = 0
        for _ in range(LAYERS):
            dfa.dfa_forward(q, k, v, cfg, out=o, stream=ctx.stream)
            n += dfa.last_launch_count()
        return n

    total_ms, launches, clocks = ctx.timed(step, steps, warmup)
    ms = total_ms / steps
    _, tc, _ = peaks()
    tf = flop_per_unit(W, R) * H * LAYERS * CONFIG5_IMAGES / (ms / 1e3) / 1e12
    res = {"value": CONFIG5_IMAGES / (ms / 1e3), "unit": "images/s", "ms_per_step": ms, "tflops": tf,
           "tensor_peak_frac": tf / tc, "gpu_launches": launches, "clocks": clocks, "dtype": "bf16",
           "scaling": "strong", "images_per_rank": mine}
    del q, k, v
    if ctx.world > 1:
        ctx.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        full = gather_to_rank0(o, CONFIG5_IMAGES)
        e1.record(ctx.stream)
        ctx.barrier()
        gt, = ctx.max_over_ranks(e0.elapsed_time(e1))
        gbytes = (CONFIG5_IMAGES - mine) * N_TOK * H * D * 2 if ctx.rank == 0 else 0
        res["gather"] = {"ms": gt, "bytes_to_rank0": gbytes, "GBps": gbytes / (gt / 1e3) / 1e9 if gbytes else None,
                         "how": "grouped ncclSend/ncclRecv of each shard's final-layer output to rank 0"}
        del full
    return res


def gather_config2(ctx, o, batch):
    torch = ctx.torch
    from paper_2403_09195_b200.dist import gather_to_rank0

    ctx.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ctx.stream)
    gathered = gather_to_rank0(o, batch * ctx.world)
    e1.record(ctx.stream)
    ctx.barrier()
    gt, = ctx.max_over_ranks(e0.elapsed_time(e1))
    gbytes = o.numel() * o.element_size() * (ctx.world - 1)
    del gathered
    return {"ms": gt, "bytes_to_rank0": gbytes, "GBps": gbytes / (gt / 1e3) / 1e9,
            "how": "grouped ncclSend/ncclRecv of each shard's output to rank 0 (paper_2403_09195_b200.dist)"}


def run_b200(args):
    ctx = Ctx(args)
    wl = args.workload
    if wl == "config2":
        res = wl_config2(ctx, args.steps, args.warmup, args.batch, with_e2e=not args.quick)
        out = res.pop("_out")
        if ctx.world > 1:
            res["gather"] = gather_config2(ctx, out, args.batch)
        del out
    elif wl == "config1":
        res = wl_config1(ctx, args.steps * 4, args.warmup)
    elif wl == "config3":
        res = wl_config3(ctx, args.steps, args.warmup, args.batch)
    elif wl == "config4":
        res = wl_config4(ctx, args.steps, args.warmup)
    elif wl == "lse":
        res = wl_lse(ctx, args.steps, args.warmup)
    else:
        res = wl_config5(ctx, max(3, args.steps // 10), args.warmup)
    extras = None
    if wl == "config2" and ctx.world == 1 and not args.quick and not args.no_extras:
        ctx.torch.cuda.empty_cache()
        # Order: lightest thermal load first.  Measured (scripts/micro/frows_after.py,
        # order_effect.py): after the config-3 graph sweep (up to 19 GB of rotating
        # inputs) the backward runs 24% and the multi-head layer 18% slower for the
        # rest of the process, and after config 4's compute-bound cells the LSE set
        # runs under sw_power_cap -- so those rows are timed before them.
        extras = {"config1": wl_config1(ctx, 256, 64)}
        ctx.torch.cuda.empty_cache()
        extras["f_rows"] = wl_frows(ctx, 20, 3)
        ctx.torch.cuda.empty_cache()
        extras["lse"] = wl_lse(ctx, 20, 3)
        time.sleep(3)  # let the board's power / temperature settle before the compute-bound cells
        extras["config4"] = wl_config4(ctx, 20, 3)
        ctx.torch.cuda.empty_cache()
        extras["config3"] = {"rows": [{k: v for k, v in wl_config3(ctx, 40, 5, b).items()
                                       if k in ("batch", "value", "ms_per_step", "tflops", "tensor_peak_frac",
                                                "clocks", "rotating_sets")}
                                      for b in (1, 2, 4, 8, 16, 32, 64, 128, 256)]}
    ctx.sampler.close()
    if ctx.rank == 0:
        emit(args, ctx.world, res, extras)
    if ctx.world > 1:
        ctx.dist.destroy_process_group()
    return 0


def emit(args, world, res, extras):
    line = {
        "metric": METRIC, "value": res["value"], "unit": res["unit"], "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
        "scaling": res.get("scaling", "weak"), "vs_baseline": None, "dtype": res.get("dtype", "bf16"),
        "data": "synthetic (torch.randn, per-rank seed; random inputs, no checkpoint needed)",
        "config": workload_config(args.workload, args, args.batch),
    }
    for key in ("tflops", "tensor_peak_frac", "roofline", "e2e", "gpu_launches", "clocks", "gather", "rows",
                "branches", "AI_fused", "images_per_rank", "us_per_call", "rotating_sets", "launches_per_call"):
        if key in res:
            line[key] = res[key]
    if "e2e" not in line:
        line["e2e"] = None
    if extras:
        line["extras"] = extras
    if world == 1 and not args.no_cpu_baseline and not args.quick:
        imgs, cores, kind, sample = cpu_reference_images_per_s(args.workload)
        line["cpu_baseline"] = {"value": imgs, "unit": "images/s", "cores": cores, "kind": kind, "sample": sample,
                                **host_info()}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ stub arm
def run_stub(args):
    """CPU stand-in for the GPU step (tests of the launcher / rank plumbing on
    gloo): same rank discovery, barrier and max-over-ranks reduction, a tiny
    torch matmul as the step."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    a = torch.randn(64, 64)
    for _ in range(args.warmup):
        a @ a
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        a @ a
    t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    if world > 1:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "impl": "stub", "value": args.batch * world * args.steps / t.item(),
                          "unit": "images/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": 1e3 * t.item() / args.steps}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------------ launcher
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_under_torchrun(args, argv):
    """`bench.py --gpus N` without WORLD_SIZE: start N ranks (one process per
    GPU) under torch.distributed.run on this node and return rank 0's exit code."""
    if not args.stub and args.impl == "b200":
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} requested but only {have} CUDA device(s) are visible",
                  file=sys.stderr, flush=True)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + argv
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.run(cmd, env=env).returncode


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", choices=WORKLOADS, default="config2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="default run: skip the configs 1/3/4/lse extras")
    ap.add_argument("--quick", action="store_true", help="profiling mode: no e2e, no CPU baseline, no extras")
    ap.add_argument("--stub", action="store_true", help=argparse.SUPPRESS)  # CPU launcher tests
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch_under_torchrun(args, argv)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr, flush=True)
        return 2
    if args.stub:
        return run_stub(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
