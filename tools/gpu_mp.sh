#!/bin/bash
# mixed-precision exploration: c5 / c4 benches with mixed off / on and GEMM variants, parity tests
cd $GRAFT_REPO_ROOT
P=${Q_PREFIX:-mp}
B="python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 3"
timeout 600 $B --config c5 --mixed 1 > gpurun_out/${P}_c5_on.log 2>&1
timeout 300 python -m pytest tests -m gpu -q -x -k "test_config_full_batch_vs_oracle_samples" > gpurun_out/${P}_pytest.log 2>&1
for g in bf16x9 tf32; do LYAP_MP_GEMM=$g timeout 600 $B --config c5 --mixed 1 > gpurun_out/${P}_c5_$g.log 2>&1; done
timeout 600 $B --config c4 --mixed 1 > gpurun_out/${P}_c4_on.log 2>&1
timeout 600 $B --config c2 --mixed 1 > gpurun_out/${P}_c2_on.log 2>&1
timeout 600 $B --config c3 --mixed 1 > gpurun_out/${P}_c3_on.log 2>&1
tail -3 gpurun_out/${P}_pytest.log
