#!/bin/bash
# Session 2: warp-loop endgame (two calls per lane on a warp's last selection), register cap A/B,
# argmin row-shape parity, NCCL single-rank bench path.
mkdir -p gpurun_out/s2f
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s2f/gpu_tests.log 2>&1
tail -2 gpurun_out/s2f/gpu_tests.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 50 --no-cpu --no-e2e > gpurun_out/s2f/c4_torchrun1.json 2> gpurun_out/s2f/c4_torchrun1.err
echo "torchrun nccl: $(tail -c 300 gpurun_out/s2f/c4_torchrun1.json)"
bash scripts/gpu_abn.sh s2f "base base_mr48 default mr48" "--config c2 --steps 300|c2" "--config c3 --dist pareto --M 10000 --steps 20|c3p4" "--config c3 --dist pareto --M 100000 --steps 5|c3p5" "--config c3 --dist exponential --M 10000 --steps 20|c3e4" "--config c5 --steps 2 --warmup 3 --max-trials 16777216|c5"
