#!/bin/bash
cd $GRAFT_REPO_ROOT
python paper_2312_08201_b200/build.py > gpurun_out/r2g_build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -k "stability or full_solution" > gpurun_out/r2g_pytest.log 2>&1
tail -3 gpurun_out/r2g_pytest.log
