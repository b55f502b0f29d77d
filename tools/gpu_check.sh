# usage: bash tools/gpu_check.sh [pytest -k expr] ; runs GPU tests then short benches
K=${1:-}
if [ -n "$K" ]; then python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_gpu.log 2>&1; else python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; fi
echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
for c in ${CHUNKS:-1}; do timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --chunk $c ${BENCH_ARGS:-} > gpurun_out/bench_chunk_$c.log 2>&1; tail -1 gpurun_out/bench_chunk_$c.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['phase_ms'], d.get('depth_phases'), d['events'].get('n_pairs'))"; done
