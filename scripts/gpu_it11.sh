#!/bin/bash
mkdir -p gpurun_out
export ZS_LIB=$PWD/paper_2603_17435_b200/libzs_trace.so
for M in 1 32 256; do echo "== L8B.GateUp M=$M"; timeout 120 python scripts/trace_gemm.py L8B.GateUp $M; done > gpurun_out/trace_r02f.txt 2>&1
echo "== L8B.O M=32" >> gpurun_out/trace_r02f.txt; timeout 120 python scripts/trace_gemm.py L8B.O 32 >> gpurun_out/trace_r02f.txt 2>&1
