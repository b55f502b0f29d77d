#!/bin/bash
# Round-2 measurement pass on one B200: GPU suite (+ parity counts), bench
# lines for the configurations DESIGN §9 quotes, the reference arm, the ncu
# launch list and the blend kernels' traffic / full captures.
O=gpurun_out/r02final; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputest.log 2>&1; tail -1 $O/gputest.log
B="python bench.py --steps 30 --warmup 5"
timeout 900 $B > $O/bench_c3_softplus.json 2> $O/bench_c3_softplus.err; tail -c 300 $O/bench_c3_softplus.json
for spec in "exp:--model exponential --no-cpu-baseline" "linear:--model linear --no-cpu-baseline" \
            "blended:--model blended --no-cpu-baseline" "cnone:--chunk none --no-cpu-baseline" \
            "c128:--chunk 128 --no-cpu-baseline" "cnone_exp:--chunk none --model exponential --no-cpu-baseline --no-e2e" \
            "c4_8views:--views-per-rank 8 --no-cpu-baseline --no-e2e" "adam:--adam --no-cpu-baseline --no-e2e" \
            "det:--deterministic --no-cpu-baseline --no-e2e"; do
  n=${spec%%:*}; a=${spec#*:}
  timeout 900 $B $a > $O/bench_c3_$n.json 2> $O/bench_c3_$n.err || tail -3 $O/bench_c3_$n.err
done
timeout 900 python bench.py --steps 3 --warmup 2 --gaussians 5000000 --width 3840 --height 2160 --model blended \
  --views-per-rank 256 --no-cpu-baseline --no-e2e > $O/bench_c5_256views.json 2> $O/bench_c5.err || tail -3 $O/bench_c5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_c3_ref.json 2> $O/bench_ref.err || tail -3 $O/bench_ref.err
N="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv $N > $O/ncu_launch.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,smsp__thread_inst_executed_per_inst_executed.ratio,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:'k_blend_(fwd|bwd)$' --launch-skip 4 -c 4 --csv $N > $O/ncu_traffic.csv 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^k_blend_(fwd|bwd)$' --launch-skip 6 -c 2 -o $O/blend_full $N > $O/ncu_full.log 2>&1
echo done
