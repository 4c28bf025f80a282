#!/bin/bash
# slot groups 2 / 3 / 4 (LYAP_GROUPS) at a few total batch sizes, c2 / c4 / c5
B="python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3"
for G in 2 3 4; do for b in 1024 1536; do LYAP_GROUPS=$G timeout 300 $B --config c2 --batch $b > gpurun_out/gr_c2_G${G}_b$b.json 2>&1; done; done
for G in 2 3; do LYAP_GROUPS=$G timeout 400 $B --config c4 > gpurun_out/gr_c4_G$G.json 2>&1; done
for G in 3; do LYAP_GROUPS=$G timeout 300 $B --config c3 > gpurun_out/gr_c3_G$G.json 2>&1; done
for G in 3; do LYAP_GROUPS=$G timeout 600 python bench.py --no-cpu-baseline --no-e2e --config c5 --steps 1 --warmup 3 > gpurun_out/gr_c5_G$G.json 2>&1; done
LYAP_GROUPS=3 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gr_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gr_pytest.log
