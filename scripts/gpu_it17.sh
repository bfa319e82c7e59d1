#!/bin/bash
mkdir -p gpurun_out
AB_LAYERS=L8B.GateUp,L8B.Down AB_MS=144,192,256 bash scripts/gpu_ab.sh it17 s3x2
AB_LAYERS=L8B.GateUp AB_MS=32 bash scripts/gpu_ab.sh it17b s3x2
