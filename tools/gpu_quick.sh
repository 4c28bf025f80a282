#!/bin/bash
# quick check of the current build: GPU tests + c5/c2/c3 benches
cd $GRAFT_REPO_ROOT
P=${Q_PREFIX:-q}
python paper_2312_08201_b200/build.py > gpurun_out/${P}_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${P}_pytest.log 2>&1
B="python bench.py --no-cpu-baseline --steps 3 --warmup 3"
for c in c5 c2 c3 c4; do timeout 600 $B --config $c > gpurun_out/${P}_bench_$c.log 2>&1; done
tail -2 gpurun_out/${P}_pytest.log
