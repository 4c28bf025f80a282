#!/bin/bash
# one ncu --set full capture of the tcgen05 K1 GEMM (and of the VERIFY DMMA GEMM) inside a c5 step
cd $GRAFT_REPO_ROOT
P=${1:-nu}
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
   -k regex:"k1_umma_persistent|k1_dgemm" -s 40 -c 2 -o gpurun_out/${P}_c5_full \
   python tools/profile_step.py c5 > gpurun_out/${P}_ncu_full.log 2>&1
echo "rc=$?" >> gpurun_out/${P}_ncu_full.log
