#!/bin/bash
# A/B of variant libraries: quick exactness check per variant, then alternating timings.
#   usage: gpu_ab.sh TAG variant1 variant2 ...   (variants = libzs_<name>.so; "base" = libzs.so)
TAG=$1; shift
mkdir -p gpurun_out
libof() { if [ "$1" = base ]; then echo $PWD/paper_2603_17435_b200/libzs.so; else echo $PWD/paper_2603_17435_b200/libzs_$1.so; fi; }
for v in "$@"; do
  echo "== $v" >> gpurun_out/ab_${TAG}_check.txt
  ZS_LIB=$(libof $v) timeout 240 python scripts/quick_check.py >> gpurun_out/ab_${TAG}_check.txt 2>&1
done
for i in 1 2; do
  for v in base "$@"; do
    ZS_LIB=$(libof $v) timeout 200 python scripts/exp_flags.py ${AB_LAYERS:-L8B.GateUp,L8B.Down} 0 ${AB_MS:-1,32} | sed "s/^{/{\"v\": \"$v\", /" >> gpurun_out/ab_${TAG}.jsonl 2>&1
  done
done
grep -c OK gpurun_out/ab_${TAG}_check.txt
