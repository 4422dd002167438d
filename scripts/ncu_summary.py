#!/usr/bin/env python3
"""Summarise an ncu capture (--set full) and a launch list into profiles/.

    python scripts/ncu_summary.py TAG REP.ncu-rep LAUNCHES.csv [WORKLOAD_KEY]

Writes profiles/TAG_ncu.md (key metrics of the attention kernel + launch
shares) and merges {WORKLOAD_KEY: dram bytes per launch} into
profiles/ncu_traffic.json (read by bench.py for roofline.traffic)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active % (active cycles)"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe % of peak"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe % of peak"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "occupancy limit (registers), CTAs/SM"),
    ("launch__occupancy_limit_shared_mem", "occupancy limit (smem), CTAs/SM"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    return [(dict(zip(h, r)), dict(zip(h, units))) for r in rows[2:]]


def to_bytes(val, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(val.replace(",", "")) * mult


def main():
    tag, rep, launches = sys.argv[1:4]
    key = sys.argv[4] if len(sys.argv) > 4 else "config2_B64_h6_w512_r2"
    lines = [f"# ncu summary `{tag}`", "", f"source: `{os.path.basename(rep)}` (ncu --set full --clock-control none), "
             f"launch list `{os.path.basename(launches)}`", ""]
    traffic = None
    for d, u in raw(rep):
        name = d.get("Kernel Name", "?")
        lines += [f"## kernel `{name[:100]}`", "", "| metric | value | unit |", "|---|---|---|"]
        for k, label in KEYS:
            if k in d:
                lines.append(f"| {label} (`{k}`) | {d[k]} | {u.get(k, '')} |")
        if "dram__bytes_read.sum" in d:
            traffic = to_bytes(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"]) + to_bytes(
                d["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
            lines.append(f"| DRAM read+write per launch | {traffic:.4g} | byte |")
        lines.append("")
    # launch shares
    with open(launches) as f:
        rows = [r for r in csv.DictReader(l for l in f if not l.startswith("==")) if
                r.get("Metric Name") == "gpu__time_duration.sum"]
    tot = {}
    for r in rows:
        nm = r["Kernel Name"].split("(")[0][:80]
        tot.setdefault(nm, []).append(float(r["Metric Value"].replace(",", "")))
    allsum = sum(sum(v) for v in tot.values())
    lines += ["## launch list (cold-cache, serialised; compare shares)", "", "| kernel | launches | mean ns | share |",
              "|---|---|---|---|"]
    for nm, v in sorted(tot.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{nm}` | {len(v)} | {sum(v) / len(v):.0f} | {sum(v) / allsum:.1%} |")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if traffic is not None:
        p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        cur = json.load(open(p)) if os.path.exists(p) else {}
        cur[key] = traffic
        json.dump(cur, open(p, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
