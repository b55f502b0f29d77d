set -x
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
for c in 128 none; do timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --chunk $c > gpurun_out/bench_chunk_$c.log 2>&1; tail -1 gpurun_out/bench_chunk_$c.log | cut -c1-1500; done
