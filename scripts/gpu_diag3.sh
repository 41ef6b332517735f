#!/bin/bash
mkdir -p gpurun_out/diag
timeout 300 python scripts/diag_host.py 2>&1 | tee gpurun_out/diag/host.txt
