#!/bin/bash
# The GPU test suite against the bounds-checked library variant (device
# asserts at the blend kernels' ring / batch / sequence indices, NXS_CHECK in
# csrc/nxs_internal.cuh).  compute-sanitizer is not available on this pool.
# build first: python -m paper_2603_02887_b200.build --variant=checks -DNXS_CHECKS
NXS_LIB=paper_2603_02887_b200/lib/libnxs_checks.so timeout 2400 python -m pytest tests -m gpu -q \
  -p no:cacheprovider > gpurun_out/checks_gputest.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/checks_gputest.log
