#!/bin/bash
# Blend-kernel counters at C3 (Mode G softplus, Mode X softplus): lane
# utilisation, pipe mix, issue activity, plus one --set full capture each.
# usage: bash tools/ncu_blend.sh TAG
set -x
T=${1:-r02}
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/${T}_bench_plain.json 2> gpurun_out/${T}_bench_plain.err || exit 1
M=smsp__thread_inst_executed_per_inst_executed.ratio,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_xu.sum,sm__inst_executed_pipe_lsu.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,smsp__thread_inst_executed_pred_on.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:'^k_blend_(fwd|bwd)$' --launch-skip 4 -c 4 --csv $B > gpurun_out/${T}_ncu_g.csv 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:'k_blend_(fwd|bwd)_x' --launch-skip 4 -c 4 --csv $B --chunk none > gpurun_out/${T}_ncu_x.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'^k_blend_(fwd|bwd)$' --launch-skip 6 -c 2 -o gpurun_out/${T}_blend_full $B > gpurun_out/${T}_ncu_full.log 2>&1
echo done
