#!/bin/bash
# mixed-precision knobs on c5 / c4: coarse space, eta, UMMA tile
cd $GRAFT_REPO_ROOT
P=${Q_PREFIX:-mx}
B="python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 3"
timeout 300 python -m pytest tests -m gpu -q -x -k "mixed" > gpurun_out/${P}_pytest.log 2>&1
timeout 600 $B --config c5 --coarse 0 > gpurun_out/${P}_c5_coarse0.log 2>&1
timeout 600 $B --config c5 --mixed-eta 1e-3 > gpurun_out/${P}_c5_eta3.log 2>&1
timeout 600 $B --config c5 --mixed-eta 1e-5 > gpurun_out/${P}_c5_eta5.log 2>&1
LYAP_UM_BN=128 timeout 600 $B --config c5 > gpurun_out/${P}_c5_bn128.log 2>&1
timeout 600 $B --config c4 --coarse 0 > gpurun_out/${P}_c4_coarse0.log 2>&1
tail -3 gpurun_out/${P}_pytest.log
