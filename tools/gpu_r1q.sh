#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/aa_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/aa_pytest.log
timeout 900 python bench.py > gpurun_out/aa_bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/aa_bench_default.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/aa_bench_torchrun.log 2>&1; echo "rc=$?" >> gpurun_out/aa_bench_torchrun.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 --cpu-seconds 10 > gpurun_out/aa_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/aa_bench_ref.log
