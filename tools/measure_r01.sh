set -x
B="timeout 400 python bench.py"
$B > gpurun_out/b_softplus.json 2> gpurun_out/b_softplus.err
$B --model exponential --no-e2e --no-cpu-baseline > gpurun_out/b_exp.json 2>/dev/null
$B --model linear --no-e2e --no-cpu-baseline > gpurun_out/b_linear.json 2>/dev/null
$B --model blended --no-e2e --no-cpu-baseline > gpurun_out/b_blended.json 2>/dev/null
$B --views-per-rank 8 --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/b_c4.json 2>/dev/null
$B --gaussians 5000000 --width 3840 --height 2160 --model blended --views-per-rank 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b_c5.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum --clock-control none -k regex:'k_blend_(fwd|bwd)$' -c 4 --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_traffic.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_blend_bwd --launch-skip 3 -c 1 -o gpurun_out/bwd_full2 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bwd2.log 2>&1
echo done
