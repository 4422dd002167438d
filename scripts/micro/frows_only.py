"""bench.py's f_rows workload alone (fresh process), twice."""
import argparse, json, sys
sys.path.insert(0, ".")
import bench
args = argparse.Namespace(gpus=1, steps=20, warmup=3, batch=64, impl="b200", workload="config2", no_cpu_baseline=True,
                          no_extras=False, quick=True, stub=False)
ctx = bench.Ctx(args)
for _ in range(2):
    r = bench.wl_frows(ctx, 20, 3)
    print({k: round(v["ms"], 4) for k, v in r.items()}, r["backward"]["clocks"]["reasons"])
ctx.sampler.close()
