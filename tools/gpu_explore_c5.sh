#!/bin/bash
# exploration: per-v GMRES iteration counts (T_d vs pair-block preconditioner) and tile-shared
# projection dims on c5 / c2 (tools/explore/tile_galerkin.py)
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 900 python tools/explore/tile_galerkin.py c5 2x2x2x2 16 gmres cuda low,high,mid,mixed,p80 > gpurun_out/x_c5_gmres.log 2>&1
timeout 1500 python tools/explore/tile_galerkin.py c5 2x2x2x2 16 galerkin cuda low,mid,high,mixed >> gpurun_out/x_c5_tiles16.log 2>&1
timeout 900 python tools/explore/tile_galerkin.py c2 8x8 16 minres cuda mixed,high >> gpurun_out/x_c2_minres.log 2>&1
timeout 1500 python tools/explore/tile_galerkin.py c5 4x4x4x4 64 galerkin cuda high,mid >> gpurun_out/x_c5_tiles256.log 2>&1
tail -5 gpurun_out/x_*.log
