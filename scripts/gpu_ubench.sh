#!/bin/bash
cd scripts/ubench
for m in 0 1 3; do for cfg in "8 4" "16 4"; do set -- $cfg; ./round $m $1 $2 2000; done; done
