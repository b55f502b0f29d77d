#!/bin/bash
# Quick GPU check of the exact/chunked orders after a K3x/K4x change.
T=${1:-qx}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_c3.py tests/test_gpu_fuzz.py -q -x -p no:cacheprovider \
  -k "exact or chunk or none or 128 or progressive or fuzz" > gpurun_out/${T}_tests.log 2>&1
tail -1 gpurun_out/${T}_tests.log
