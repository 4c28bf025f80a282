#!/bin/bash
# full GPU tests + bench lines (c5, c4, c2, c3) + ncu launch list of a c5 step + the small-shard batch experiment
cd $GRAFT_REPO_ROOT
P=${Q_PREFIX:-q4}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${P}_pytest.log 2>&1
tail -2 gpurun_out/${P}_pytest.log
B="python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3"
for c in c5 c4 c2 c3; do timeout 300 $B --config $c > gpurun_out/${P}_$c.log 2>&1; done
python tools/bench_summary.py gpurun_out/${P}_c5.log gpurun_out/${P}_c4.log gpurun_out/${P}_c2.log gpurun_out/${P}_c3.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
   --clock-control none -c 4000 --csv --log-file gpurun_out/${P}_launches_c5.csv \
   python tools/profile_step.py c5 > gpurun_out/${P}_ncu1.log 2>&1
python tools/ncu_summary.py gpurun_out/${P}_launches_c5.csv > gpurun_out/${P}_kernels.txt 2>&1
head -14 gpurun_out/${P}_kernels.txt
bash tools/gpu_smallshard.sh
