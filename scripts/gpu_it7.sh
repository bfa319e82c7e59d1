#!/bin/bash
mkdir -p gpurun_out
AB_LAYERS=L8B.GateUp,L8B.Down,L8B.QKV,L8B.O AB_MS=1,32 bash scripts/gpu_ab.sh it7a lsel rt32 rt32lsel incr all3
AB_LAYERS=L8B.GateUp,L8B.Down AB_MS=64,96,128 bash scripts/gpu_ab.sh it7b s3x3 s3x2
