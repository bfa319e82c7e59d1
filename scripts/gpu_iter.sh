#!/bin/bash
# One iteration on the GPU box: parity subset, timing knobs, variant libraries, one ncu capture
# of the fused kernel.   usage: gpu_iter.sh TAG [variant.so ...]
TAG=${1:-it}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_${TAG}.log 2>&1
timeout 300 python scripts/exp_flags.py L8B.GateUp,L8B.O,L8B.Down 0,1,8,9,12,13,14 1,32 > gpurun_out/flags_${TAG}.jsonl 2>&1
timeout 300 python scripts/exp_flags.py L8B.GateUp 0 1,32 --dist realistic > gpurun_out/flags_real_${TAG}.jsonl 2>&1
for v in "$@"; do
  ZS_LIB=$PWD/paper_2603_17435_b200/$v timeout 300 python scripts/exp_flags.py L8B.GateUp,L8B.Down 0,8 1,32 > gpurun_out/flags_${TAG}_${v%.so}.jsonl 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:zipgemm -s 4 -c 1 -f -o gpurun_out/prof_${TAG} python bench.py --steps 5 --warmup 2 --m 32 --no-extras --no-cpu-baseline > gpurun_out/prof_${TAG}.log 2>&1
ls -la gpurun_out
