#!/bin/bash
mkdir -p gpurun_out/div
timeout 1500 ./scripts/ubench/divcheck > gpurun_out/div/divcheck.txt 2>&1; echo "rc=$?" >> gpurun_out/div/divcheck.txt
cat gpurun_out/div/divcheck.txt
timeout 900 python -m pytest tests -m gpu -x -q -k "argmin or table1" > gpurun_out/div/tests.log 2>&1; tail -2 gpurun_out/div/tests.log
timeout 300 python bench.py --config p1 --steps 100 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; r=json.loads(sys.stdin.read()); print('p1', r['value'], r['roofline']['frac'])"
timeout 300 python bench.py --config p1 --M 64 --steps 100 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; r=json.loads(sys.stdin.read()); print('p1 M64', r['value'], r['roofline']['frac'])"
