mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_v8a.log 2>&1
timeout 300 python scripts/exp_flags.py L8B.GateUp,L8B.O,L8B.Down 0,1,8,12,13 1,32 > gpurun_out/flags_v8a.jsonl 2>&1
timeout 300 python scripts/exp_flags.py L8B.GateUp 0 1,32 --dist realistic > gpurun_out/flags_real_v8a.jsonl 2>&1
ZS_LIB=$PWD/paper_2603_17435_b200/libzs_trace.so timeout 120 python scripts/trace_gemm.py L8B.GateUp 32 > gpurun_out/trace_v8a.txt 2>&1
ZS_LIB=$PWD/paper_2603_17435_b200/libzs_trace.so timeout 120 python scripts/trace_gemm.py L8B.GateUp 32 8 > gpurun_out/trace_v8a_nohbm.txt 2>&1
