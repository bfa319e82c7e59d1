#!/bin/bash
# Validation of the 3-stage split at M = 129..256 (ZS_SPLIT3=2 default): GPU tests, smoke, bench,
# large-M sweep.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02i.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r02i.log 2>&1
timeout 300 python bench.py > gpurun_out/bench_r02i.json 2> gpurun_out/bench_r02i.err
timeout 600 python scripts/sweep_gemm.py --layers L8B.GateUp,L8B.Down --ms 129,192,256 --modes fused,decoupled --cublas --graph-steps 10 > gpurun_out/sweep_large_r02i.jsonl 2>&1
timeout 300 python scripts/sweep_gemm.py --layers L8B.GateUp --ms 96,128,144,160,192,224,256 --cublas --graph-steps 10 > gpurun_out/sweep_m_r02i.jsonl 2>&1
