#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/af_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/af_pytest.log
for md in 0 256 512; do
  timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --config c5 --max-dim $md > gpurun_out/af_${md}_c5.log 2>&1
done
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --config c4 --max-dim 320 > gpurun_out/af_320_c4.log 2>&1
