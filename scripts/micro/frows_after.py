"""f_rows after each of the default bench's earlier workloads, to find which
one leaves the backward slower."""
import argparse, sys
sys.path.insert(0, ".")
import bench
args = argparse.Namespace(gpus=1, steps=200, warmup=5, batch=64, impl="b200", workload="config2", no_cpu_baseline=True,
                          no_extras=False, quick=False, stub=False)
ctx = bench.Ctx(args)
def fr(tag):
    r = bench.wl_frows(ctx, 20, 3)
    print(tag, {k: round(v["ms"], 4) for k, v in r.items()}, flush=True)
fr("start")
res = bench.wl_config2(ctx, 200, 5, 64, with_e2e=True); res.pop("_out"); ctx.torch.cuda.empty_cache()
fr("after config2+e2e")
bench.wl_config1(ctx, 256, 64)
fr("after config1")
for b in (1, 2, 4, 8, 16, 32, 64, 128, 256):
    bench.wl_config3(ctx, 40, 5, b)
ctx.torch.cuda.empty_cache()
fr("after config3 sweep")
ctx.sampler.close()
