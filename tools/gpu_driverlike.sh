#!/bin/bash
# the two invocations the driver makes at round end, with its round-1 arguments: our arm and the reference arm
cd $GRAFT_REPO_ROOT
P=${EV_PREFIX:-ev7}
( time timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/${P}_driver_ours.log 2>&1
( time timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/${P}_driver_reference.log 2>&1
timeout 900 python bench.py > gpurun_out/${P}_bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_bench_default.log
tail -4 gpurun_out/${P}_driver_ours.log | cut -c1-300; tail -4 gpurun_out/${P}_driver_reference.log | cut -c1-600
