#!/bin/bash
# Quick GPU check after a kernel change: Mode G parity subset + bench lines.
# usage: bash tools/quick_gpu.sh TAG [extra bench args]
T=${1:-q}; shift
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_c3.py -q -x -p no:cacheprovider \
  -k "c1_forward or c1_backward or progressive or fused or device_sized or c3" > gpurun_out/${T}_tests.log 2>&1
tail -2 gpurun_out/${T}_tests.log
for m in softplus exponential; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --model $m "$@" > gpurun_out/${T}_bench_$m.json 2> gpurun_out/${T}_bench_$m.err
  python -c "import json;d=json.load(open('gpurun_out/${T}_bench_$m.json'));print('$m', d['value'], d['ms_per_step'], d['phase_ms'].get('blend_fwd'), d['phase_ms'].get('blend_bwd'), d['roofline']['blend_fp32'])"
done
