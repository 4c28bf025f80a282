#!/bin/bash
# exploration: two-level (coarse-space) preconditioner vs TSVD-SMW vs pair, c5 / c4 / c2
cd $GRAFT_REPO_ROOT
timeout 1500 python tools/explore/tsvd_prec.py c5 64,128,200 cuda > gpurun_out/x2l_c5.log 2>&1
timeout 900 python tools/explore/tsvd_prec.py c4 64,128,200 cuda > gpurun_out/x2l_c4.log 2>&1
timeout 600 python tools/explore/tsvd_prec.py c2 64,128,200 cuda > gpurun_out/x2l_c2.log 2>&1
