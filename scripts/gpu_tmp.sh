mkdir -p gpurun_out
for i in 1 2; do
timeout 300 python scripts/exp_flags.py L8B.GateUp,L8B.Down 0 1,32,128 > gpurun_out/ab4_cur_$i.jsonl 2>&1
ZS_LIB=$PWD/paper_2603_17435_b200/libzs_v8.so timeout 300 python scripts/exp_flags.py L8B.GateUp,L8B.Down 0 1,32 > gpurun_out/ab4_v8_$i.jsonl 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "forced or integer or one_hot or oracle" > gpurun_out/pytest_v9f.log 2>&1
