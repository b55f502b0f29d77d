for nb in 5 6 4; do
  sed -i "s/__launch_bounds__(BWD_THREADS, [0-9])/__launch_bounds__(BWD_THREADS, $nb)/" paper_2603_02887_b200/csrc/blend_bwd.cu
  python -c "from paper_2603_02887_b200 import build as b; b.build(force=True, verbose=True)" > gpurun_out/sw_build_$nb.log 2>&1
  grep -A3 "Compiling entry function '_ZN3nxs11k_blend_bwdILi6ELb0" gpurun_out/sw_build_$nb.log | tail -2
  for m in softplus exponential; do timeout 200 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --model $m | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$nb', '$m', d['value'], d['ms_per_step'], d['phase_ms']['blend_bwd'])"; done
done
