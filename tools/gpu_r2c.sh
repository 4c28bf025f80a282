#!/bin/bash
cd $GRAFT_REPO_ROOT
python paper_2312_08201_b200/build.py > gpurun_out/r2c_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -k "extended_krylov" > gpurun_out/r2c_pytest_ek.log 2>&1
timeout 600 python tools/explore/c5_applies.py c5 > gpurun_out/r2c_applies_c5.log 2>&1
for b in 296 444 888; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --batch $b --steps 2 --warmup 3 > gpurun_out/r2c_c5_b$b.log 2>&1; done
for m in 256 512; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --max-dim $m --steps 2 --warmup 3 > gpurun_out/r2c_c5_m$m.log 2>&1; done
timeout 600 python bench.py --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/r2c_c5_default.log 2>&1
