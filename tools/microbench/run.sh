set -x
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/mb_clocks.csv &
SMI=$!
./tools/microbench/fp64_peak > gpurun_out/fp64_peak.txt 2>&1
python tools/microbench/dgemm_peak.py > gpurun_out/dgemm_peak.txt 2>&1
kill $SMI
nproc > gpurun_out/box_cpu.txt; lscpu >> gpurun_out/box_cpu.txt
