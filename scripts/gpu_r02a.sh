mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_r02a.txt
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02a.log 2>&1
timeout 300 python bench.py --steps 200 --warmup 10 > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err
timeout 300 python scripts/exp_flags.py L8B.GateUp,L8B.O 0,1,4,5 1,32 > gpurun_out/flags_r02a.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:zipgemm -s 4 -c 1 -f -o gpurun_out/prof_r02a python bench.py --steps 5 --warmup 2 --m 32 --no-extras --no-cpu-baseline > gpurun_out/prof_r02a.log 2>&1
ls -la gpurun_out
