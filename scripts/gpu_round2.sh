#!/bin/bash
mkdir -p gpurun_out/r2
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
tail -5 gpurun_out/gpu_tests.log
for M in 64 256 1024; do timeout 300 python bench.py --config p1 --M $M --steps 100 --no-cpu --no-e2e > gpurun_out/r2/p1_$M.json 2>&1; done
timeout 300 python bench.py --config c4 --rule argmin --steps 20 --no-cpu --no-e2e > gpurun_out/r2/c4_argmin.json 2>&1
timeout 300 python bench.py --steps 500 > gpurun_out/r2/c4.json 2>&1
# multi-rank dry run (2 ranks share this GPU over gloo): exercises sharding, C1-C3
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config c2 --steps 50 --no-cpu --no-e2e --dist-backend gloo > gpurun_out/r2/c2_2ranks.json 2> gpurun_out/r2/c2_2ranks.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --K 262144 --steps 20 --no-cpu --dist-backend gloo > gpurun_out/r2/c4_2ranks.json 2> gpurun_out/r2/c4_2ranks.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r2/ref.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select_rows -s 3 -c 1 -o gpurun_out/prof_c4_v2 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_c4_v2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select_shared -s 3 -c 1 -o gpurun_out/prof_c3u python bench.py --config c3 --dist uniform --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_c3u.log 2>&1
