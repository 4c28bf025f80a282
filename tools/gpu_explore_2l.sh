#!/bin/bash
# exploration: coarse spaces for the two-level preconditioner (harmonic Ritz from seed solves vs TSVD)
cd $GRAFT_REPO_ROOT
timeout 1500 python tools/explore/ritz_coarse.py c5 8 cuda > gpurun_out/xr_c5.log 2>&1
timeout 900 python tools/explore/ritz_coarse.py c4 8 cuda > gpurun_out/xr_c4.log 2>&1
