#!/bin/bash
# Final-state check + f4 workload sweep with the final kernel.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02e.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r02e.log 2>&1
timeout 900 python scripts/sweep_gemm.py --layers L70B.QKV,L70B.O,L70B.GateUp,L70B.Down,L70B.QKV.w8,L70B.O.w8,L70B.GateUp.w8,L70B.Down.w8,Q32B.QKV,Q32B.O,Q32B.GateUp,Q32B.Down,G3-27B.QKV,G3-27B.O,G3-27B.GateUp,G3-27B.Down,Q2.5-7B.QKV,Q2.5-7B.O,Q2.5-7B.GateUp,Q2.5-7B.Down,L8B.LMHead --ms 1,32 --cublas --graph-steps 10 > gpurun_out/sweep_models_r02e.jsonl 2>&1
ls -la gpurun_out
