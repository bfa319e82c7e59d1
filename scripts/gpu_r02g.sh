#!/bin/bash
# Characterisation of the final kernel: M sweep on 8B GateUp and the heavy-tailed case per layer
# (CUDA graphs of 10 launches with PDL, cuBLAS beside).
mkdir -p gpurun_out
timeout 900 python scripts/sweep_gemm.py --layers L8B.GateUp --ms 1,2,4,8,16,32,48,64,96,128,192,256 --cublas --graph-steps 10 > gpurun_out/sweep_m_r02g.jsonl 2>&1
timeout 600 python scripts/sweep_gemm.py --layers L8B.QKV,L8B.O,L8B.GateUp,L8B.Down --ms 1,32 --dist realistic --graph-steps 10 > gpurun_out/sweep_real_r02g.jsonl 2>&1
timeout 600 python scripts/sweep_gemm.py --layers L8B.QKV,L8B.O,L8B.GateUp,L8B.Down --ms 1,32 --graph-steps 10 > gpurun_out/sweep_gauss_r02g.jsonl 2>&1
