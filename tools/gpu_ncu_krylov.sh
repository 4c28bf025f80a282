#!/bin/bash
# ncu --set full of the HBM-bound Krylov kernels inside a c5 trace_batch (one launch each, mid-batch)
cd $GRAFT_REPO_ROOT
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
   -k regex:"k_dots|k_upd|k_prec|k_xcomb|k1_gen16" -s 500 -c 5 -o gpurun_out/krylov_c5 -f \
   python tools/profile_step.py c5 > gpurun_out/krylov_ncu.log 2>&1
echo "rc=$?"
ncu -i gpurun_out/krylov_c5.ncu-rep --page raw --csv > gpurun_out/krylov_c5_raw.csv 2>/dev/null
wc -c gpurun_out/krylov_c5_raw.csv
