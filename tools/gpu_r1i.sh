#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
LYAP_NVCC_EXTRA="-DSMALL_BK=32" python paper_2312_08201_b200/build.py --force > gpurun_out/p_build.log 2>&1
for c in c2 c3; do timeout 400 $B --config $c > gpurun_out/p_bk32_$c.log 2>&1; done
python paper_2312_08201_b200/build.py --force >> gpurun_out/p_build.log 2>&1
