#!/bin/bash
# Round-2 evidence of HEAD: GPU tests, smoke, bench line, launch list, one ncu capture.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_r02d.txt
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02d.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r02d.log 2>&1
timeout 300 python bench.py --steps 200 --warmup 10 > gpurun_out/bench_r02d.json 2> gpurun_out/bench_r02d.err
timeout 300 python scripts/exp_flags.py L8B.GateUp,L8B.Down,L8B.QKV,L8B.O 0,1 1,32 > gpurun_out/flags_r02d.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02d.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_r02d.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:zipgemm -s 4 -c 1 -f -o gpurun_out/prof_r02d python bench.py --steps 5 --warmup 3 --m 32 --no-extras --no-cpu-baseline > gpurun_out/prof_r02d.log 2>&1

timeout 300 python scripts/decomp_bench.py > gpurun_out/decomp_r02d.jsonl 2>&1
timeout 600 python scripts/sweep_gemm.py --layers L8B.QKV,L8B.O,L8B.GateUp,L8B.Down --ms 1,32,128,256 --cublas --graph-steps 1 > gpurun_out/sweep_small_r02d.jsonl 2>&1
timeout 300 python scripts/sweep_gemm.py --layers L8B.GateUp --ms 1,32 --dist realistic --graph-steps 1 > gpurun_out/sweep_real_r02d.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decompress -s 2 -c 1 -f -o gpurun_out/prof_decomp_r02d python scripts/decomp_bench.py --iters 5 --layers L8B.GateUp > gpurun_out/prof_decomp_r02d.log 2>&1
timeout 600 python scripts/sweep_gemm.py --layers L8B.GateUp,L8B.Down,L8B.QKV --ms 129,256,512,2048 --modes fused,decoupled --cublas --graph-steps 1 > gpurun_out/sweep_large_r02d.jsonl 2>&1
ls -la gpurun_out
