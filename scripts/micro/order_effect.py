"""LSE set and config-4 compute-bound cells before / after the config-3 batch
sweep (the default bench used to run the sweep first)."""
import argparse, sys
sys.path.insert(0, ".")
import bench
args = argparse.Namespace(gpus=1, steps=200, warmup=5, batch=64, impl="b200", workload="config2", no_cpu_baseline=True,
                          no_extras=False, quick=False, stub=False)
ctx = bench.Ctx(args)
def probe(tag):
    l = bench.wl_lse(ctx, 20, 3)
    c4 = bench.wl_config4(ctx, 20, 3)
    cells = {f"{r['w']}:{r['r']}": round(r["ms"], 4) for r in c4["rows"] if (r["w"], r["r"]) in ((4096, 1), (2048, 1), (512, 2), (256, 8))}
    print(tag, "lse", round(l["ms_per_step"], 4), "per-branch", round(l["per_branch"]["ms_per_step"], 4), cells, flush=True)
probe("before config3")
for b in (1, 2, 4, 8, 16, 32, 64, 128, 256):
    bench.wl_config3(ctx, 40, 5, b)
ctx.torch.cuda.empty_cache()
probe("after config3")
ctx.sampler.close()
