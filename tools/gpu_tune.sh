#!/bin/bash
# compile-time variants of the Krylov-kernel load parallelism (rebuilt on the box), c2 + c4 bench
B="python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3"
for v in "-DLYAP_DOT_IG=32" "-DLYAP_DOT_IG=128" "-DLYAP_UPD_UNROLL=4" "-DLYAP_UPD_UNROLL=16" ""; do
  tag=$(echo "x$v" | tr -c 'A-Za-z0-9' '_')
  LYAP_NVCC_EXTRA="$v" python paper_2312_08201_b200/build.py > gpurun_out/tu_build$tag.log 2>&1 || continue
  timeout 300 $B --config c2 > gpurun_out/tu_c2$tag.json 2>&1
  timeout 400 $B --config c4 > gpurun_out/tu_c4$tag.json 2>&1
done
