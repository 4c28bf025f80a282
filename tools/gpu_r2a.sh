#!/bin/bash
# round 2: GPU tests + smoke + bench c5 (default) and c1-c4 after the pair-block preconditioner
cd $GRAFT_REPO_ROOT
python paper_2312_08201_b200/build.py > gpurun_out/r2a_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2a_bench_c5.log 2>&1
for c in c1 c2 c3 c4; do timeout 600 python bench.py --config $c --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/r2a_bench_$c.log 2>&1; done
tail -3 gpurun_out/r2a_pytest.log
