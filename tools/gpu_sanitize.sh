#!/bin/bash
cd "$(dirname "$0")/.."
timeout 300 python tools/sanitize_driver.py > gpurun_out/s_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python tools/sanitize_driver.py > gpurun_out/s_memcheck.log 2>&1
echo "rc=$?" >> gpurun_out/s_memcheck.log
