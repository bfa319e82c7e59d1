mkdir -p gpurun_out
for i in 1 2; do
timeout 300 python scripts/exp_flags.py L8B.GateUp 0,12 1,32 > gpurun_out/ab3_cur_$i.jsonl 2>&1
ZS_LIB=$PWD/paper_2603_17435_b200/libzs_x8.so timeout 300 python scripts/exp_flags.py L8B.GateUp 0,12 1,32 > gpurun_out/ab3_x8_$i.jsonl 2>&1
ZS_LIB=$PWD/paper_2603_17435_b200/libzs_v8.so timeout 300 python scripts/exp_flags.py L8B.GateUp 0,12 1,32 > gpurun_out/ab3_v8_$i.jsonl 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "forced or integer or one_hot" > gpurun_out/pytest_v9e.log 2>&1
