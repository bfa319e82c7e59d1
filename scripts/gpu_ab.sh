#!/bin/bash
# A/B of variant libraries: parity subset per variant, then alternating timings.
#   usage: gpu_ab.sh TAG variant1 variant2 ...   (variants = libzs_<name>.so; "base" = libzs.so)
TAG=$1; shift
mkdir -p gpurun_out
libof() { if [ "$1" = base ]; then echo $PWD/paper_2603_17435_b200/libzs.so; else echo $PWD/paper_2603_17435_b200/libzs_$1.so; fi; }
for v in "$@"; do
  ZS_LIB=$(libof $v) timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "forced or integer or one_hot or oracle" > gpurun_out/ab_${TAG}_pytest_$v.log 2>&1
  echo "$v pytest rc=$?" >> gpurun_out/ab_${TAG}_summary.txt
  tail -1 gpurun_out/ab_${TAG}_pytest_$v.log >> gpurun_out/ab_${TAG}_summary.txt
done
for i in 1 2; do
  for v in base "$@"; do
    ZS_LIB=$(libof $v) timeout 300 python scripts/exp_flags.py ${AB_LAYERS:-L8B.GateUp,L8B.Down} 0 ${AB_MS:-1,32} | sed "s/^{/{\"v\": \"$v\", /" >> gpurun_out/ab_${TAG}.jsonl 2>&1
  done
done
cat gpurun_out/ab_${TAG}_summary.txt
