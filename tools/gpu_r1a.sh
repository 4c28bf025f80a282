#!/bin/bash
# round-1 first GPU pass: smoke, parity tests, short benches
cd "$(dirname "$0")/.."
nvidia-smi > gpurun_out/a_smi.txt 2>&1
nproc > gpurun_out/a_cpu.txt; lscpu >> gpurun_out/a_cpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/a_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/a_smoke.log
timeout 900 python -m pytest tests -m gpu -x -q -k "not c4 and not c5" > gpurun_out/a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/a_pytest.log
for c in c1 c2 c3; do
  timeout 600 python bench.py --config $c --steps 2 --warmup 1 --cpu-seconds 5 > gpurun_out/a_bench_$c.log 2>&1; echo "rc=$?" >> gpurun_out/a_bench_$c.log
done
