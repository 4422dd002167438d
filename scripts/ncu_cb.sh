mkdir -p gpurun_out
for s in "2048 1" "512 1"; do set -- $s
timeout 300 ncu --set full --clock-control none --import-source on -k regex:dfa_sm100 -s 2 -c 1 -o gpurun_out/prof_cb_$1_$2 -f python scripts/micro/fwd_once.py $1 $2 32 > gpurun_out/prof_cb_$1_$2.log 2>&1
done
ls -la gpurun_out | tail
