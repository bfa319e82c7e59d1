#!/bin/bash
mkdir -p gpurun_out
AB_LAYERS=L8B.GateUp,L8B.Down,L8B.QKV,L8B.O AB_MS=1,32 bash scripts/gpu_ab.sh it15 hyb1k hyb4k
