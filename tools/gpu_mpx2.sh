#!/bin/bash
# verify-GEMM tile, coarse space under mixed precision, per-rank batches at N = 8
cd $GRAFT_REPO_ROOT
P=${Q_PREFIX:-mx2}
B="python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 3"
timeout 300 python -m pytest tests -m gpu -q -x -k "mixed or test_config_full_batch_vs_oracle_samples" > gpurun_out/${P}_pytest.log 2>&1
timeout 600 $B --config c5 > gpurun_out/${P}_c5.log 2>&1
LYAP_VER_BN=64 timeout 600 $B --config c5 > gpurun_out/${P}_c5_ver64.log 2>&1
timeout 600 $B --config c5 --coarse 0 > gpurun_out/${P}_c5_coarse0.log 2>&1
timeout 600 $B --config c5 --emulate-rank 0/8 > gpurun_out/${P}_emu8.log 2>&1
timeout 600 $B --config c5 --emulate-rank 0/8 --batch 256 > gpurun_out/${P}_emu8_b256.log 2>&1
timeout 600 $B --config c5 --emulate-rank 0/4 > gpurun_out/${P}_emu4.log 2>&1
timeout 600 $B --config c4 > gpurun_out/${P}_c4.log 2>&1
tail -3 gpurun_out/${P}_pytest.log
