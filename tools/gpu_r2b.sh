#!/bin/bash
cd $GRAFT_REPO_ROOT
python paper_2312_08201_b200/build.py > gpurun_out/r2b_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -k "extended_krylov" > gpurun_out/r2b_pytest_ek.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2b_pytest.log 2>&1
for c in c5 c4 c2; do timeout 900 python tools/explore/recycle_sweep.py $c > gpurun_out/r2b_rec_$c.log 2>&1; done
tail -3 gpurun_out/r2b_pytest.log
