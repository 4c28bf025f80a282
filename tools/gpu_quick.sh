#!/bin/bash
cd $GRAFT_REPO_ROOT
python paper_2312_08201_b200/build.py > gpurun_out/fu_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/fu_pytest.log 2>&1
B="python bench.py --no-cpu-baseline --steps 3 --warmup 3"
for c in c5 c2 c1; do timeout 600 $B --config $c > gpurun_out/fu_bench_$c.log 2>&1; done
LYAP_GROUPS=1 timeout 600 $B --config c5 > gpurun_out/fu_bench_c5_G1.log 2>&1
tail -2 gpurun_out/fu_pytest.log
