#!/bin/bash
# Team-size sweep (GPUAR_TEAM) against the device's model choice, per shared-vector config.
out=gpurun_out/${1:-team}; mkdir -p $out
val() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('%.4g(g=%s)' % (d['value'], (d.get('trials') or {}).get('team')))" $1 2>/dev/null || echo fail; }
run() {  # name "args" teams...
  name=$1; args=$2; shift 2
  line="$name"
  for g in "$@"; do
    if [ $g = model ]; then GPUAR_TEAM= timeout 300 python bench.py $args --no-cpu --no-e2e > $out/${name}_$g.json 2>&1
    else GPUAR_TEAM=$g timeout 300 python bench.py $args --no-cpu --no-e2e > $out/${name}_$g.json 2>&1; fi
    line="$line | $g: $(val $out/${name}_$g.json)"
  done
  echo "$line"
}
run c2 "--config c2 --steps 300" model 8 16 32 model 16
run c3p3 "--config c3 --dist pareto --M 1000 --steps 20" model 4 8 16 32
run c3e3 "--config c3 --dist exponential --M 1000 --steps 20" model 1 2 4
run c3e5 "--config c3 --dist exponential --M 100000 --steps 20" model 1 2 4 8
run c3u4 "--config c3 --dist uniform --M 10000 --steps 20" model 1 2
run c1 "--config c1 --steps 300" model 1 2 4
