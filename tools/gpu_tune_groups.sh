#!/bin/bash
cd $GRAFT_REPO_ROOT
python paper_2312_08201_b200/build.py > gpurun_out/g_build.log 2>&1
B="python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 3"
LYAP_GROUPS=1 timeout 600 $B > gpurun_out/g_c5_G1.log 2>&1
LYAP_GROUPS=1 timeout 600 $B --batch 888 > gpurun_out/g_c5_G1_b888.log 2>&1
LYAP_GROUPS=1 timeout 600 $B --batch 444 > gpurun_out/g_c5_G1_b444.log 2>&1
LYAP_GROUPS=3 timeout 600 $B --batch 888 > gpurun_out/g_c5_G3_b888.log 2>&1
for c in c2 c3 c4; do LYAP_GROUPS=1 timeout 600 $B --config $c > gpurun_out/g_${c}_G1.log 2>&1; done
LYAP_GROUPS=1 timeout 600 $B --emulate-rank 0/8 > gpurun_out/g_emu8_G1.log 2>&1
LYAP_GROUPS=1 timeout 600 $B --emulate-rank 0/8 --batch 256 > gpurun_out/g_emu8_G1_b256.log 2>&1
timeout 600 $B --emulate-rank 0/8 --batch 256 > gpurun_out/g_emu8_G2_b256.log 2>&1
