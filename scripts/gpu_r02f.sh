#!/bin/bash
# Final evidence of the committed state: GPU tests, smoke, bench line, launch list, ncu capture.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_r02f.txt
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02f.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r02f.log 2>&1
timeout 300 python bench.py > gpurun_out/bench_r02f.json 2> gpurun_out/bench_r02f.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r02f.json 2> gpurun_out/bench_ref_r02f.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02f.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_r02f.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:zipgemm -s 4 -c 1 -f -o gpurun_out/prof_r02f python bench.py --steps 5 --warmup 3 --m 32 --no-extras --no-cpu-baseline > gpurun_out/prof_r02f.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decompress -s 2 -c 1 -f -o gpurun_out/prof_decomp_r02f python scripts/decomp_bench.py --iters 5 --layers L8B.GateUp > gpurun_out/prof_decomp_r02f.log 2>&1
ls -la gpurun_out
