#!/bin/bash
cd "$(dirname "$0")/.."
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
for ce in 256 512; do
  LYAP_NVCC_EXTRA="-DLYAP_RED_CE=$ce" python paper_2312_08201_b200/build.py --force > gpurun_out/ac_build_$ce.log 2>&1
  timeout 900 python -m pytest tests -m gpu -q -x -k "random_instances or config_full" > gpurun_out/ac_pytest_$ce.log 2>&1; echo "rc=$?" >> gpurun_out/ac_pytest_$ce.log
  for c in c2 c3 c4; do timeout 400 $B --config $c > gpurun_out/ac_${ce}_$c.log 2>&1; done
  timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --config c5 > gpurun_out/ac_${ce}_c5.log 2>&1
done
python paper_2312_08201_b200/build.py --force >> gpurun_out/ac_build_256.log 2>&1
