#!/bin/bash
# Session 2: s1 (SSA loop) re-measurement: the session-start build vs the current one, interleaved.
mkdir -p gpurun_out/s2i
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,temperature.gpu --format=csv > gpurun_out/s2i/smi.txt 2>&1
cat gpurun_out/s2i/smi.txt
bash scripts/gpu_abn.sh s2i "start default" "--config s1 --steps 20|s1" "--config s1 --steps 20|s1b"
