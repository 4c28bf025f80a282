#!/bin/bash
# quick check of a Krylov-kernel change: mixed-precision tests, c5/c4 bench lines, ncu launch list of a c5 step
cd $GRAFT_REPO_ROOT
P=${Q_PREFIX:-q2}
timeout 900 python -m pytest tests -m gpu -q -x -k "mixed or config_full or sharded or random_instances" > gpurun_out/${P}_pytest.log 2>&1
tail -2 gpurun_out/${P}_pytest.log
B="python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3"
timeout 300 $B --config c5 > gpurun_out/${P}_c5.log 2>&1
timeout 300 $B --config c4 > gpurun_out/${P}_c4.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
   --clock-control none -c 4000 --csv --log-file gpurun_out/${P}_launches_c5.csv \
   python tools/profile_step.py c5 > gpurun_out/${P}_ncu1.log 2>&1
python tools/bench_summary.py gpurun_out/${P}_c5.log gpurun_out/${P}_c4.log 2>/dev/null
