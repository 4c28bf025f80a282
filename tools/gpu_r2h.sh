#!/bin/bash
cd $GRAFT_REPO_ROOT
python paper_2312_08201_b200/build.py > gpurun_out/r2h_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k "qlin or extended_krylov or full_solution" > gpurun_out/r2h_pytest.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2h_pytest_all.log 2>&1
tail -3 gpurun_out/r2h_pytest_all.log
