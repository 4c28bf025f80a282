#!/bin/bash
# recycle-space refinement study: tests touching recycling, then c5/c4 benches per rounds setting
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu -k "recycl or forced or restart" > gpurun_out/rf_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/rf_tests.log
for r in 1 2 3; do
  LYAP_RECYCLE_ROUNDS=$r timeout 600 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/rf_c5_r$r.json 2> gpurun_out/rf_c5_r$r.err
done
for r in 1 2; do
  LYAP_RECYCLE_ROUNDS=$r timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --recycle 32 --no-cpu-baseline --no-e2e > gpurun_out/rf_c4_r$r.json 2> gpurun_out/rf_c4_r$r.err
done
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --recycle 0 --no-cpu-baseline --no-e2e > gpurun_out/rf_c4_r0.json 2> gpurun_out/rf_c4_r0.err
