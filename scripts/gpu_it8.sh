#!/bin/bash
mkdir -p gpurun_out
AB_LAYERS=L8B.GateUp,L8B.Down,L8B.QKV AB_MS=1,32 bash scripts/gpu_ab.sh it8 lutmix lpred h64 lpmix h64lp
for v in base h64; do
  L=$PWD/paper_2603_17435_b200/libzs_$v.so; [ $v = base ] && L=$PWD/paper_2603_17435_b200/libzs.so
  ZS_LIB=$L timeout 200 python scripts/decomp_bench.py --layers L8B.GateUp,L8B.Down | sed "s/^{/{\"v\": \"$v\", /" >> gpurun_out/decomp_it8.jsonl 2>&1
done
