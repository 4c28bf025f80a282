#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q -k "extended_krylov" > gpurun_out/z2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/z2_pytest.log
