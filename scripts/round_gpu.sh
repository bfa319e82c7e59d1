#!/bin/bash
# One GPU session for the round's evidence (run under gpurun): tests, smoke, bench line,
# sweeps, launch list + ncu full capture.  Outputs land in gpurun_out/ (copied to profiles/).
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_${TAG}.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_${TAG}.log 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 600 python scripts/decomp_bench.py --iters 100 > gpurun_out/decomp_${TAG}.jsonl 2>&1
timeout 900 python scripts/sweep_gemm.py --layers L8B.GateUp,L8B.QKV,L8B.O,L8B.Down --ms 1,8,32,64,128 --cublas > gpurun_out/sweep_small_${TAG}.jsonl 2>&1
bash scripts/ncu_profile.sh ${TAG} 32 > gpurun_out/ncu_script_${TAG}.log 2>&1
ls -la gpurun_out
