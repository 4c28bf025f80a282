#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python tools/explore/tsvd_prec.py c5 50,100,200,400 cuda > gpurun_out/r2d_tsvd_c5.log 2>&1
timeout 600 python tools/explore/tsvd_prec.py c2 25,50,100,200 cuda > gpurun_out/r2d_tsvd_c2.log 2>&1
timeout 900 python tools/explore/tsvd_prec.py c4 50,100,200,400 cuda > gpurun_out/r2d_tsvd_c4.log 2>&1
