#!/bin/bash
mkdir -p gpurun_out
AB_LAYERS=L8B.QKV,L8B.O,L70B.O.w8,L70B.GateUp.w8 AB_MS=1,32 bash scripts/gpu_ab.sh it3 ws ilppws ilppws2 ctl32
AB_LAYERS=L8B.GateUp AB_MS=32,128,256 bash scripts/gpu_ab.sh it3b ilppws ilppws2
