mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_v9a.log 2>&1
timeout 300 python scripts/exp_flags.py L8B.GateUp,L8B.O 0 1,32,128 > gpurun_out/flags_v9a.jsonl 2>&1
timeout 1200 python scripts/sweep_gemm.py --layers L8B.GateUp,L8B.Down,L8B.QKV,L8B.O --ms 129,192,256,384,512,1024,2048 --modes fused,decoupled --cublas --iters 30 > gpurun_out/sweep_large_v9a.jsonl 2>&1
