B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/small_plain.json 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_depth|k_key32_hist|k_phase_select|k_bin_scatter|k_bin_sort|k_project_ranks|k_emit_tiles|k_seg_sort_warp|k_chain|k_call_init' --launch-skip 30 -c 10 -o gpurun_out/small2_full $B > gpurun_out/small2_ncu.log 2>&1
tail -2 gpurun_out/small2_ncu.log
