#!/bin/bash
# Round-2 evidence on the current build (one gpurun call):
#   tests + smoke; the default bench (c5, with cpu_baseline and e2e); c1-c4 benches; per-rank
#   emulation of the 2/4/8-GPU strong split of c5; the EK demo (f1); the ncu launch list of a c5 step
#   and one full ncu capture of the c5 K1 GEMM.   Output: gpurun_out/ev_*  (summarised into profiles/)
cd "$(dirname "$0")/.."
P=${EV_PREFIX:-ev}
python paper_2312_08201_b200/build.py > gpurun_out/${P}_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${P}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${P}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_smoke.log
timeout 900 python bench.py > gpurun_out/${P}_bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_bench_default.log
for c in c1 c2 c3 c4; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${P}_bench_$c.log 2>&1; done
for r in 2 4 8; do timeout 600 python bench.py --emulate-rank 0/$r --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${P}_emu_$r.log 2>&1; done
timeout 900 python tools/ek_demo.py c3 c5 > gpurun_out/${P}_ek_demo.log 2>&1
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/${P}_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
   --clock-control none -k regex:"^(k_|k1_)" -s 26000 -c 1600 --csv --log-file gpurun_out/${P}_launches_c5.csv $CMD > gpurun_out/${P}_ncu1.log 2>&1
echo "launch rc=$?" >> gpurun_out/${P}_plain.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k1_dgemm -s 60 -c 2 \
    -o gpurun_out/${P}_k1full_c5 $CMD > gpurun_out/${P}_ncu2.log 2>&1
echo "full rc=$?" >> gpurun_out/${P}_plain.log
