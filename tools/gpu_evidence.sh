#!/bin/bash
# Round-2 evidence on the current build (one gpurun call):
#   tests + smoke; the default bench (c5, with cpu_baseline and e2e); c1-c4 benches; c5 FP64-only;
#   per-rank emulation of the 2/4/8-GPU strong split of c5; the EK demo (f1); the reference arm;
#   the tcgen05 GEMM microbenchmark; the ncu launch list of one c5 trace_batch (profiling window) and
#   one ncu --set full capture of the tcgen05 K1 GEMM and the VERIFY DMMA GEMM.
#   Output: gpurun_out/<prefix>_*  (summarised into profiles/ by tools/make_summary_r02.py)
cd "$(dirname "$0")/.."
P=${EV_PREFIX:-ev}
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${P}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${P}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_smoke.log
timeout 900 python bench.py > gpurun_out/${P}_bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_bench_default.log
for c in c1 c2 c3 c4; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${P}_bench_$c.log 2>&1; done
timeout 600 python bench.py --config c5 --mixed 0 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${P}_bench_c5_fp64.log 2>&1
for r in 2 4 8; do timeout 600 python bench.py --emulate-rank 0/$r --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${P}_emu_$r.log 2>&1; done
timeout 900 python tools/ek_demo.py c3 c5 > gpurun_out/${P}_ek_demo.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${P}_reference.log 2>&1
(cd tools/microbench && timeout 120 ./umma_tf32x3 4096 4736 4000 && timeout 120 ./umma_tf32x3 4096 4864 4000) > gpurun_out/${P}_umma_micro.log 2>&1
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
   --clock-control none -c 4000 --csv --log-file gpurun_out/${P}_launches_c5.csv \
   python tools/profile_step.py c5 > gpurun_out/${P}_ncu1.log 2>&1
echo "launch rc=$?" >> gpurun_out/${P}_ncu1.log
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
   -k regex:"k1_umma_persistent|k1_dgemm" -s 40 -c 2 -o gpurun_out/${P}_k1full_c5 \
   python tools/profile_step.py c5 > gpurun_out/${P}_ncu2.log 2>&1
echo "full rc=$?" >> gpurun_out/${P}_ncu2.log
