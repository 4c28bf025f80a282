#!/bin/bash
# blocked back-substitution: gpu tests, c2/c5/c4 bench, c2 launch list of the engine kernels
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/bs_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/bs_pytest.log
B="python bench.py --no-cpu-baseline --no-e2e"
timeout 400 $B --config c2 --steps 3 --warmup 3 > gpurun_out/bs_c2.json 2>&1
timeout 400 $B --config c4 --steps 3 --warmup 3 > gpurun_out/bs_c4.json 2>&1
timeout 900 $B --config c5 --steps 2 --warmup 3 > gpurun_out/bs_c5.json 2>&1
CMD="python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed \
   --clock-control none -k regex:"^(k_|k1_)" -s 3000 -c 1400 --csv --log-file gpurun_out/bs_kern_c2.csv $CMD > gpurun_out/bs_ncu1.log 2>&1
echo "ncu rc=$?" >> gpurun_out/bs_ncu1.log
