#!/bin/bash
# A/B kernel variants: bench each lib/libnxs_<v>.so (plus the default) at C3.
# usage: bash tools/ab_bench.sh TAG "v1 v2 ..." [extra bench args]
T=$1; V=$2; shift 2
for v in default $V; do
  if [ $v = default ]; then L=paper_2603_02887_b200/lib/libnxs.so; else L=paper_2603_02887_b200/lib/libnxs_$v.so; fi
  for rep in 1 2; do
    NXS_LIB=$L timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline "$@" > gpurun_out/${T}_$v.json 2> gpurun_out/${T}_$v.err
    python -c "import json;d=json.load(open('gpurun_out/${T}_$v.json'));print('%-10s'%'$v', d['value'], d['ms_per_step'], 'fwd',d['phase_ms'].get('blend_fwd'), 'bwd',d['phase_ms'].get('blend_bwd'), 'frac', d['roofline']['blend_fp32']['frac_of_derived_peak'])" || tail -3 gpurun_out/${T}_$v.err
  done
done
