#!/bin/bash
# Session 2: compute-sanitizer over every kernel after the session-2 kernel changes, and
# 2-rank torchrun dry runs (gloo on one GPU) of the c2 / c4 / s1 bench paths.
bash scripts/gpu_sanitize.sh
mkdir -p gpurun_out/s2n
for spec in "--config c2 --steps 50|c2" "--K 262144 --steps 20|c4" "--config s1 --steps 5|s1" "--config c5 --steps 2 --warmup 3 --max-trials 16777216|c5"; do
  args=${spec%%|*}; name=${spec##*|}
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 $args --no-cpu --no-e2e --dist-backend gloo > gpurun_out/s2n/${name}_2ranks.json 2> gpurun_out/s2n/${name}_2ranks.err
  echo "$name 2 ranks rc=$? $(tail -c 400 gpurun_out/s2n/${name}_2ranks.json | head -c 400)"
done
