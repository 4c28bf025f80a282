#!/bin/bash
# restored M1 / sharded tests, then a sweep of the refinement-cycle reduction mixed_eta and the restart length on c5 / c4
cd $GRAFT_REPO_ROOT
export LYAP_MP_ORDER=0
timeout 900 python -m pytest tests/test_gpu_sweep.py -m gpu -q -x > gpurun_out/eta_pytest.log 2>&1
tail -3 gpurun_out/eta_pytest.log
EV_PREFIX=eta bash tools/gpu_sweep.sh \
 "c5 eta 1e-4||--config c5" \
 "c5 eta 3e-5||--config c5 --mixed-eta 3e-5" \
 "c5 eta 1e-5||--config c5 --mixed-eta 1e-5" \
 "c5 eta 1e-6||--config c5 --mixed-eta 1e-6" \
 "c5 eta 1e-3||--config c5 --mixed-eta 1e-3" \
 "c5 eta 1e-5 md 512||--config c5 --mixed-eta 1e-5 --max-dim 512" \
 "c5 eta 1e-4 md 256||--config c5 --max-dim 256" \
 "c4 eta 1e-4||--config c4" \
 "c4 eta 1e-5||--config c4 --mixed-eta 1e-5" \
 "c4 eta 1e-6||--config c4 --mixed-eta 1e-6"
cat gpurun_out/eta_sweep.log
