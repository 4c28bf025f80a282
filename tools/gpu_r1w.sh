#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/ah_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ah_pytest.log
timeout 900 python bench.py --config c5 --steps 1 --warmup 1 --cpu-seconds 30 > gpurun_out/ah_c5.log 2>&1; echo "rc=$?" >> gpurun_out/ah_c5.log
timeout 900 python bench.py > gpurun_out/ah_default.log 2>&1; echo "rc=$?" >> gpurun_out/ah_default.log
