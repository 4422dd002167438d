mkdir -p gpurun_out
./scripts/micro/mufu_bench > gpurun_out/mufu.txt 2>&1
python scripts/trace_timeline.py run --w 512 --r 2 > gpurun_out/trace_512_2.txt 2>&1
python scripts/trace_timeline.py run --w 2048 --r 1 > gpurun_out/trace_2048_1.txt 2>&1
cat gpurun_out/mufu.txt gpurun_out/trace_512_2.txt gpurun_out/trace_2048_1.txt
