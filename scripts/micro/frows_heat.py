"""Does a long run of heavy workloads slow the f_rows afterwards?  f_rows,
then config4 + lse (as in the default bench), then f_rows again; GPU
temperature / memory clock printed between."""
import argparse, subprocess, sys
sys.path.insert(0, ".")
import bench
def smi():
    return subprocess.run(["nvidia-smi", "--query-gpu=temperature.gpu,temperature.memory,clocks.sm,clocks.mem,power.draw,clocks_throttle_reasons.active",
                           "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
args = argparse.Namespace(gpus=1, steps=20, warmup=3, batch=64, impl="b200", workload="config2", no_cpu_baseline=True,
                          no_extras=False, quick=True, stub=False)
ctx = bench.Ctx(args)
r = bench.wl_frows(ctx, 20, 3); print("cold f_rows", {k: round(v["ms"], 4) for k, v in r.items()}, smi(), flush=True)
bench.wl_config4(ctx, 20, 3); bench.wl_lse(ctx, 20, 3); ctx.torch.cuda.empty_cache()
print("after config4+lse", smi(), flush=True)
r = bench.wl_frows(ctx, 20, 3); print("hot f_rows", {k: round(v["ms"], 4) for k, v in r.items()}, smi(), flush=True)
import time; time.sleep(20)
print("after 20 s idle", smi(), flush=True)
r = bench.wl_frows(ctx, 20, 3); print("rested f_rows", {k: round(v["ms"], 4) for k, v in r.items()}, smi(), flush=True)
ctx.sampler.close()
