#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/exp_flags.py L8B.GateUp,L8B.O 0,4,8,1,5 1,32,256 > gpurun_out/flags_r02h.jsonl 2>&1
