#!/bin/bash
# A/B of the mixed-precision K1 launch order (LYAP_MP_ORDER) and the co-resident VERIFY GEMM configurations on c5
cd $GRAFT_REPO_ROOT
P=${Q_PREFIX:-ord}
B="python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 --config c5"
LYAP_MP_ORDER=0 timeout 300 $B > gpurun_out/${P}_o0.log 2>&1
timeout 300 $B > gpurun_out/${P}_o1_v2.log 2>&1
LYAP_VER_CFG=0 timeout 300 $B > gpurun_out/${P}_o1_v0.log 2>&1
LYAP_UM_ST=3 LYAP_VER_CFG=0 timeout 300 $B > gpurun_out/${P}_o1_um3_v0.log 2>&1
LYAP_UM_ST=3 LYAP_VER_CFG=2 timeout 300 $B > gpurun_out/${P}_o1_um3_v2.log 2>&1
timeout 300 $B --config c4 > gpurun_out/${P}_c4_o1.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/${P}_pytest.log 2>&1
tail -2 gpurun_out/${P}_pytest.log
