#!/bin/bash
# Session 2 close: the driver's round-end sequence on HEAD (GPU tests, smoke, default bench).
mkdir -p gpurun_out/s2zj
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s2zj/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/s2zj/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2zj/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/s2zj/bench.json 2> gpurun_out/s2zj/bench.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/s2zj/bench.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks'], d['e2e']['value'], d['gpu_launches'])"
timeout 600 python bench.py --impl reference > gpurun_out/s2zj/ref.json 2>&1; echo "ref rc=$?"; tail -c 300 gpurun_out/s2zj/ref.json
