#!/bin/bash
mkdir -p gpurun_out
for v in base w24s1 w20s1; do
  L=$PWD/paper_2603_17435_b200/libzs_$v.so; [ $v = base ] && L=$PWD/paper_2603_17435_b200/libzs.so
  ZS_LIB=$L timeout 200 python scripts/decomp_bench.py --layers L8B.GateUp,L8B.Down | sed "s/^{/{\"v\": \"$v\", /" >> gpurun_out/decomp_it2.jsonl 2>&1
done
AB_MS=1,32 bash scripts/gpu_ab.sh it2 ws il pp ilpp ildppp ilppws dp
