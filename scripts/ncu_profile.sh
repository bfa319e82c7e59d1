#!/bin/bash
# Run on the GPU box (gpurun).  Produces the launch list and one full capture of the
# top kernel under gpurun_out/.  Numbers printed under ncu are never bench values.
set -x
TAG=${1:-r01}
M=${2:-32}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 20 --warmup 3 --m $M --no-extras --no-cpu-baseline > gpurun_out/launches_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:zipgemm -s 4 -c 1 -f -o gpurun_out/prof_${TAG} \
    python bench.py --steps 5 --warmup 2 --m $M --no-extras --no-cpu-baseline > gpurun_out/prof_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decompress -s 2 -c 1 -f -o gpurun_out/prof_decomp_${TAG} \
    python scripts/decomp_bench.py --iters 5 --layers L8B.GateUp > gpurun_out/prof_decomp_${TAG}.log 2>&1
ls -la gpurun_out
