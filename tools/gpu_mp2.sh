#!/bin/bash
# mixed precision: new GPU tests + ncu launch list of a c5 MP step (all kernels, cuBLAS included)
cd $GRAFT_REPO_ROOT
P=${Q_PREFIX:-mp2}
timeout 600 python -m pytest tests -m gpu -q -x -k "mixed_precision_configs" > gpurun_out/${P}_pytest.log 2>&1
CMD="python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
   --clock-control none -s 62000 -c 4000 --csv --log-file gpurun_out/${P}_launches_c5.csv $CMD > gpurun_out/${P}_ncu1.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${P}_ncu1.log
tail -3 gpurun_out/${P}_pytest.log
