"""The reference's benchmark harness (bench.hpp) on the B200 path.

A caller of the hot path (`bench_attention`, bench.hpp:125-133),
restated with the same names, fields, CSV columns and error behaviour so
reference and B200 reports diff cleanly:

  BenchConfigEntry / BenchRow / BenchReport / SweepConfig   bench.hpp:16-47
  time_samples_ms (warm-up, coarse-clock guard)              bench.hpp:55-77
  percentile                                                 bench.hpp:79-83
  bench_attention (dense one-shot vs dilated, per batch)     bench.hpp:88-156
  run_sweep (config-major, batch-minor rows)                 bench.hpp:159-171
  bench_csv_header / bench_csv_row / write_bench_csv         bench.hpp:173-198
  SweepConfig.from_json (sweep_config_from_json)             bench.hpp:200-231
  spearman_rank_correlation                                  bench.hpp:235-276

B200 differences, by design: a "pass" is ONE batched device launch over
[batch, N, h, d] (the reference loops batch x heads on the host), samples are
device times from CUDA events, and the dense baseline is the same kernel at
(w, r) = (N, 1) -- full softmax attention, the reference's `naive_attention`.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from typing import Callable, List

from . import AttentionConfig, ConfigError, ContractError, DfaError, _fmt_double, dfa_forward, flop_count


class BenchmarkError(DfaError):
    """attnkit::benchmark_error (common.hpp:28-30)."""


@dataclass
class BenchConfigEntry:
    id: str
    attn: AttentionConfig


@dataclass
class BenchRow:
    id: str = ""
    n: int = 0
    w: int = 0
    r: int = 0
    h: int = 0
    d: int = 0
    kernel: str = "naive"
    batch: int = 0
    median_ms: float = 0.0
    p10_ms: float = 0.0
    p90_ms: float = 0.0
    dense_mults: int = 0
    dilated_mults: int = 0
    measured_speedup: float = 0.0


@dataclass
class BenchReport:
    rows: List[BenchRow] = field(default_factory=list)
    workers: int = 1
    dtype: str = "f32"


@dataclass
class SweepConfig:
    configs: List[BenchConfigEntry] = field(default_factory=list)
    batch_sizes: List[int] = field(default_factory=lambda: [1])
    repeats: int = 5
    workers: int = 1
    seed: int = 0
    quantize_ns: int = 0

    @staticmethod
    def from_json(j) -> "SweepConfig":
        """bench.hpp:200-231 sweep_config_from_json; missing keys / unknown
        kernels raise ConfigError like the reference's config_error."""
        if isinstance(j, str):
            j = json.loads(j)
        s = SweepConfig()
        try:
            s.repeats = int(j.get("repeats", s.repeats))
            s.workers = int(j.get("workers", s.workers))
            s.seed = int(j.get("seed", s.seed))
            s.quantize_ns = int(j.get("quantize_ns", s.quantize_ns))
            if "batch_sizes" in j:
                s.batch_sizes = [int(b) for b in j["batch_sizes"]]
            for e in j.get("configs", []):
                h = int(e.get("h", 1))
                r = int(e["r"])
                kernel = e.get("kernel", "naive")
                if kernel not in ("naive", "tiled"):
                    raise ConfigError(f"bench: unknown kernel {kernel}")
                attn = AttentionConfig(int(e["N"]), int(e["w"]), r, h, int(e["d"]),
                                       AttentionConfig.spread_offsets(h, r), kernel=kernel,
                                       tile_size=int(e.get("tile_size", 8)))
                attn.validate()
                s.configs.append(BenchConfigEntry(e.get("id", f"config{len(s.configs)}"), attn))
        except KeyError as ex:
            raise ConfigError(f"bench config: missing key {ex}") from None
        return s


def time_samples_ms(fn: Callable[[], None], repeats: int, quantize_ns: int = 0, warmup: int = 3) -> List[float]:
    """bench.hpp:55-77 with device time: `warmup` unrecorded runs, then one
    CUDA-event sample per run; samples floored to quantize_ns (test hook) must
    land on >= 3 distinct values or the clock is reported too coarse."""
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(repeats)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    ns = [int(round(a.elapsed_time(b) * 1e6)) for a, b in ev]
    if quantize_ns > 0:
        ns = [t - t % quantize_ns for t in ns]
    if len(set(ns)) < 3:
        raise BenchmarkError(f"timer resolution too coarse: {repeats} repeats landed on only {len(set(ns))} "
                             "distinct tick values; lengthen the workload or use a finer clock")
    return [t / 1e6 for t in ns]


def percentile(sorted_samples: List[float], pct: float) -> float:
    """bench.hpp:79-83: nearest rank, idx = llround(pct / 100 * (n - 1))."""
    k = len(sorted_samples) - 1
    idx = int(math.floor(pct / 100.0 * k + 0.5))
    return sorted_samples[idx]


def _kernel_name(cfg: AttentionConfig) -> str:
    return cfg.kernel if isinstance(cfg.kernel, str) else ("tiled" if cfg.kernel else "naive")


def bench_attention(entry: BenchConfigEntry, batch_sizes: List[int], repeats: int, workers: int = 1,
                    seed: int = 0, quantize_ns: int = 0, dtype: str = "f32") -> BenchReport:
    """bench.hpp:88-156: dense baseline vs the dilated pipeline on identical
    random inputs, one row per batch size."""
    import torch

    if repeats < 3:
        raise BenchmarkError(f"need at least 3 repeats, got {repeats}")
    cfg = entry.attn
    cfg.validate()
    fc = flop_count(cfg)
    report = BenchReport(workers=workers, dtype=dtype)
    td = torch.float32 if dtype == "f32" else torch.bfloat16
    dense = AttentionConfig(cfg.seq_len, cfg.seq_len, 1, cfg.num_heads, cfg.head_dim, [0] * cfg.num_heads,
                            scale_scores=cfg.scale_scores)
    g = torch.Generator(device="cuda").manual_seed(seed ^ 0x9E3779B97F4A7C15)
    for batch in batch_sizes:
        if batch < 1:
            raise ConfigError(f"bench: batch size must be positive, got {batch}")
        shape = (batch, cfg.seq_len, cfg.num_heads, cfg.head_dim)
        q, k, v = (torch.randn(shape, generator=g, device="cuda", dtype=td) for _ in range(3))
        o = torch.empty_like(q)
        dense_ms = sorted(time_samples_ms(lambda: dfa_forward(q, k, v, dense, out=o), repeats, quantize_ns))
        dil_ms = sorted(time_samples_ms(lambda: dfa_forward(q, k, v, cfg, out=o), repeats, quantize_ns))
        med = percentile(dil_ms, 50)
        report.rows.append(BenchRow(
            id=entry.id, n=cfg.seq_len, w=cfg.segment_len, r=cfg.interval, h=cfg.num_heads, d=cfg.head_dim,
            kernel=_kernel_name(cfg), batch=batch, median_ms=med, p10_ms=percentile(dil_ms, 10),
            p90_ms=percentile(dil_ms, 90), dense_mults=fc.dense_mults, dilated_mults=fc.dilated_mults,
            measured_speedup=percentile(dense_ms, 50) / med))
    return report


def run_sweep(sweep: SweepConfig, dtype: str = "f32") -> BenchReport:
    """bench.hpp:159-171: configs in file order, batch sizes within each."""
    report = BenchReport(workers=sweep.workers, dtype=dtype)
    for salt, entry in enumerate(sweep.configs):
        part = bench_attention(entry, sweep.batch_sizes, sweep.repeats, sweep.workers, sweep.seed + salt,
                               sweep.quantize_ns, dtype)
        report.rows.extend(part.rows)
    return report


def bench_csv_header() -> str:
    return "id,N,w,r,h,d,kernel,batch,median_ms,p10_ms,p90_ms,dense_mults,dilated_mults,measured_speedup"


def bench_csv_row(row: BenchRow) -> str:
    return ",".join([row.id, str(row.n), str(row.w), str(row.r), str(row.h), str(row.d), row.kernel, str(row.batch),
                     _fmt_double(row.median_ms), _fmt_double(row.p10_ms), _fmt_double(row.p90_ms),
                     str(row.dense_mults), str(row.dilated_mults), _fmt_double(row.measured_speedup)])


def write_bench_csv(out, report: BenchReport) -> None:
    """bench.hpp:181-198; `out` is a path or a text stream."""
    text = bench_csv_header() + "\n" + "".join(bench_csv_row(r) + "\n" for r in report.rows)
    text += f"# workers={report.workers}\n# dtype={report.dtype}\n# flop_convention=multiplications_only\n"
    if isinstance(out, str):
        try:
            with open(out, "w") as f:
                f.write(text)
        except OSError:
            from . import TensorIOError

            raise TensorIOError(f"cannot write {out}") from None
    else:
        out.write(text)


def spearman_rank_correlation(a: List[float], b: List[float]) -> float:
    """bench.hpp:235-276: tie-averaged ranks; ContractError when undefined."""
    if len(a) != len(b) or len(a) < 2:
        raise ContractError("spearman: need two equal-length series of at least 2 points")

    def ranks(x):
        order = sorted(range(len(x)), key=lambda i: x[i])
        rank = [0.0] * len(x)
        i = 0
        while i < len(x):
            j = i
            while j + 1 < len(x) and x[order[j + 1]] == x[order[i]]:
                j += 1
            for kk in range(i, j + 1):
                rank[order[kk]] = (i + j) / 2.0 + 1.0
            i = j + 1
        return rank

    ra, rb = ranks(a), ranks(b)
    n = float(len(a))
    ma, mb = sum(ra) / n, sum(rb) / n
    cov = sum((x - ma) * (y - mb) for x, y in zip(ra, rb))
    va = sum((x - ma) ** 2 for x in ra)
    vb = sum((y - mb) ** 2 for y in rb)
    if va == 0 or vb == 0:
        raise ContractError("spearman: a series is constant, correlation undefined")
    return cov / math.sqrt(va * vb)


__all__ = ["BenchConfigEntry", "BenchRow", "BenchReport", "SweepConfig", "BenchmarkError", "time_samples_ms",
           "percentile", "bench_attention", "run_sweep", "bench_csv_header", "bench_csv_row", "write_bench_csv",
           "spearman_rank_correlation"]
