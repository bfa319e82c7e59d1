mkdir -p gpurun_out
for i in 1 2; do
timeout 300 python scripts/exp_flags.py L8B.GateUp,L8B.Down 0 1,32 > gpurun_out/ab_cur_$i.jsonl 2>&1
ZS_LIB=$PWD/paper_2603_17435_b200/libzs_v8.so timeout 300 python scripts/exp_flags.py L8B.GateUp,L8B.Down 0 1,32 > gpurun_out/ab_v8_$i.jsonl 2>&1
done
timeout 1500 python -m pytest tests/test_gpu_sanitizer.py -q > gpurun_out/pytest_sanitizer.log 2>&1
