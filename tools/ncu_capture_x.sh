#!/bin/bash
# One --set full capture of the Mode X blend kernels (K3x, K4x) at C3.
# usage: bash tools/ncu_capture_x.sh TAG
T=$1; shift
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --chunk none $@"
timeout 300 $B > gpurun_out/${T}_plain.json 2> gpurun_out/${T}_plain.err || { tail -5 gpurun_out/${T}_plain.err; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_blend_(fwd|bwd)_x' --launch-skip 6 -c 2 -o gpurun_out/${T}_full $B > gpurun_out/${T}_ncu.log 2>&1
tail -2 gpurun_out/${T}_ncu.log
