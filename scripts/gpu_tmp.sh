mkdir -p gpurun_out
timeout 300 python scripts/exp_flags.py L8B.GateUp 0,2,4,6,8,10,12,14 1,32 > gpurun_out/flags_v5b.jsonl 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "decomp or Decomp or decompress" > gpurun_out/pytest_v5b_decomp.log 2>&1
timeout 300 python scripts/decomp_bench.py --iters 50 > gpurun_out/decomp_v5b.jsonl 2>&1
