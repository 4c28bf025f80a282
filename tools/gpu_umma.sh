#!/bin/bash
# tcgen05 3xTF32 GEMM: microbench variants, mixed-precision tests, c5/c4 benches (UMMA vs cuBLAS)
cd $GRAFT_REPO_ROOT
P=${Q_PREFIX:-um}
(cd tools/microbench && timeout 120 ./umma_tf32x3 4096 4864 4000 && timeout 120 ./umma_tf32x3 2048 4608 2000) > gpurun_out/${P}_micro.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "mixed or test_config_full_batch" > gpurun_out/${P}_pytest.log 2>&1
B="python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 3"
timeout 600 $B --config c5 > gpurun_out/${P}_c5.log 2>&1
LYAP_MP_GEMM=cublas timeout 600 $B --config c5 > gpurun_out/${P}_c5_cublas.log 2>&1
timeout 600 $B --config c4 > gpurun_out/${P}_c4.log 2>&1
tail -3 gpurun_out/${P}_pytest.log
