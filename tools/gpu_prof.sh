#!/bin/bash
# ncu launch list of one whole-grid trace_batch (profiling window only): $1 = config, $2 = mixed, $3 = prefix
cd $GRAFT_REPO_ROOT
C=${1:-c5}; M=${2:--1}; P=${3:-prof}
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
   --clock-control none -c ${NCU_COUNT:-3000} --csv --log-file gpurun_out/${P}_launches_${C}.csv \
   python tools/profile_step.py $C --mixed $M > gpurun_out/${P}_${C}_prof.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${P}_${C}_prof.log
