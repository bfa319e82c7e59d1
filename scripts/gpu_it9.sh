#!/bin/bash
mkdir -p gpurun_out
L=$PWD/paper_2603_17435_b200/libzs_dstage.so
ZS_LIB=$L timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k decompress > gpurun_out/it9_pytest_dstage.log 2>&1
for i in 1 2; do
for v in base dstage; do
  L=$PWD/paper_2603_17435_b200/libzs_$v.so; [ $v = base ] && L=$PWD/paper_2603_17435_b200/libzs.so
  ZS_LIB=$L timeout 200 python scripts/decomp_bench.py --layers L8B.GateUp,L8B.Down,L8B.QKV | sed "s/^{/{\"v\": \"$v\", /" >> gpurun_out/decomp_it9.jsonl 2>&1
done
done
tail -1 gpurun_out/it9_pytest_dstage.log
