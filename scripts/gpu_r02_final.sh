#!/bin/bash
# Round-2 final evidence: GPU tests, smoke, bench (both arms), launch list, ncu capture of the headline kernel.
TAG=${1:-r02f}
OUT=gpurun_out; mkdir -p $OUT
timeout 1100 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 > $OUT/tests_$TAG.log 2>&1
echo "tests rc=$?" >> $OUT/tests_$TAG.log; tail -3 $OUT/tests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; tail -1 $OUT/smoke_$TAG.log
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref_$TAG.json 2>> $OUT/bench_$TAG.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches_$TAG.csv python bench.py --steps 10 --warmup 3 --quick > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:dfa_sm100 -s 5 -c 1 -o $OUT/prof_$TAG -f python bench.py --steps 3 --warmup 3 --quick > /dev/null 2>&1
python - <<PY
import json
d=json.load(open("$OUT/bench_$TAG.json")); r=json.load(open("$OUT/bench_ref_$TAG.json"))
print("value", d["value"], "ms", d["ms_per_step"], "frac", d["roofline"]["frac"], "e2e", d["e2e"]["value"], "clk", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
print("ref", r["value"], "ratio e2e", d["e2e"]["value"]/r["value"])
ex=d["extras"]; print("config1 us", ex["config1"]["us_per_call"], "lse ms", ex["lse"]["ms_per_step"], ex["lse"]["per_branch"]["ms_per_step"])
print({k: round(v["ms"],4) for k,v in ex["f_rows"].items()})
PY
