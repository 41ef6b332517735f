#!/bin/bash
# The one GPU-box driver (run through gpurun from the repo root):
#   bash scripts/gpu.sh <task> [args]
# Tasks (outputs under gpurun_out/<dir>):
#   tests [dir]                       pytest -m gpu (+ smoke) -> <dir>/gpu_tests.log, smoke.log
#   final [dir]                       round-end evidence: tests, smoke, every workload's bench line,
#                                     the reference arm, the c4 ncu launch list, results.md
#   sanitize                          compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over
#                                     scripts/sanitize_cases.py and tests/tail_overread_case.py -> san/
#                                     (the pool closed compute-sanitizer after r02_compute_sanitizer.md:
#                                     it now exits 86 at start-up)
#   ubench [dir]                      trial-round / Philox instruction-mix microbenchmark (scripts/ubench)
#   ncu <name> <kernel-regex> <bench args...>
#                                     one `ncu --set full` capture of the first matching launch after
#                                     warm-up -> prof_<name>.ncu-rep (summarise here: scripts/ncu_summary.py)
#   launches <name> <bench args...>   ncu launch list (gpu__time_duration, clocks unlocked) -> launches_<name>.csv
#   ab <dir> "<bench args>|<label>" ...
#                                     interleaved A/B: lib/exp_base.so (scripts/build_head.sh base) vs
#                                     the working-tree build, two repetitions each
#   abn <dir> "<lib1> <lib2> ..." "<bench args>|<label>" ...
#                                     N-way A/B of lib/exp_<lib>.so builds ("default" = libgpuar.so)
#   team-sweep [dir]                  forced team sizes (GPUAR_TEAM) against the device model's choice
#   divcheck                          exhaustive check of the argmin rule's reciprocal division (R23)
set -u
task=${1:-tests}; shift || true
val() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('%.4g' % d['value'])" $1 2>/dev/null || echo fail; }
case $task in
tests)
  out=gpurun_out/${1:-tests}; mkdir -p $out
  timeout 1500 python -m pytest tests -m gpu -q -rs > $out/gpu_tests.log 2>&1
  tail -3 $out/gpu_tests.log
  timeout 300 python __graft_entry__.py --smoke > $out/smoke.log 2>&1
  tail -1 $out/smoke.log ;;
final)
  out=gpurun_out/${1:-final}; mkdir -p $out
  bash scripts/gpu.sh tests $(basename $out)
  timeout 600 python bench.py > $out/c4.json 2> $out/c4.err
  timeout 900 python bench.py --impl reference > $out/c4_reference.json 2>&1
  timeout 300 python bench.py --config c1 --steps 300 > $out/c1.json 2>&1
  timeout 300 python bench.py --config c2 --steps 300 > $out/c2.json 2>&1
  for d in uniform exponential pareto; do for M in 1000 10000 100000; do
    timeout 300 python bench.py --config c3 --dist $d --M $M --steps 20 --no-e2e > $out/c3_${d}_$M.json 2>&1
  done; done
  timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-e2e --cpu-seconds 20 > $out/c5.json 2>&1
  timeout 300 python bench.py --config p1 --steps 100 > $out/p1.json 2>&1
  timeout 300 python bench.py --config c4 --rule argmin --steps 20 --no-e2e > $out/c4_argmin.json 2>&1
  timeout 300 python bench.py --config c2 --rule it --steps 300 --no-e2e > $out/c2_it.json 2>&1
  timeout 600 python bench.py --config s1 --steps 20 > $out/s1.json 2>&1
  timeout 120 python scripts/philox_peak.py > $out/philox_peak.txt 2>&1
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c4.csv \
    python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-it --sustain-s 0 --epochs 1 --no-stream-ceiling > $out/launches_c4.log 2>&1
  python scripts/collect_results.py $out > $out/results.md ;;
sanitize)
  out=gpurun_out/san; mkdir -p $out; rm -f $out/summary.txt
  python scripts/sanitize_cases.py > $out/plain.log 2>&1
  echo "plain rc=$? $(tail -1 $out/plain.log)" >> $out/summary.txt
  for tool in memcheck racecheck synccheck initcheck; do
    extra=""
    if [ $tool = synccheck ]; then extra="--num-cuda-barriers 65536"; fi
    for case in scripts/sanitize_cases.py tests/tail_overread_case.py; do
      log=$out/${tool}_$(basename $case .py).log
      timeout 1500 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 20 python $case > $log 2>&1
      echo "$tool $case rc=$? | $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $log | tail -1) | $(grep -E '^ok|cases ok|MISMATCH' $log | tail -1)" >> $out/summary.txt
    done
  done
  cat $out/summary.txt ;;
ubench)
  out=gpurun_out/${1:-ubench}; mkdir -p $out
  (cd scripts/ubench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o round round.cu) || exit 1
  for rep in 1 2; do for m in 0 4 3 5; do for cfg in "8 4" "16 4"; do set -- $cfg
    scripts/ubench/round $m $1 $2 2000; done; done; done > $out/ubench.txt 2>&1
  cat $out/ubench.txt ;;
ncu)
  name=$1; kre=$2; shift 2
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$kre" -s 3 -c 1 \
    -o gpurun_out/prof_$name python bench.py "$@" --steps 2 --warmup 3 --no-cpu --no-e2e --no-it --sustain-s 0 --epochs 1 --no-stream-ceiling > gpurun_out/ncu_$name.log 2>&1
  tail -5 gpurun_out/ncu_$name.log ;;
launches)
  name=$1; shift
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$name.csv \
    python bench.py "$@" --steps 5 --warmup 3 --no-cpu --no-e2e --no-it --sustain-s 0 --epochs 1 --no-stream-ceiling > gpurun_out/launches_$name.log 2>&1
  tail -2 gpurun_out/launches_$name.log ;;
ab)
  out=gpurun_out/$1; shift; mkdir -p $out
  for spec in "$@"; do
    args=${spec%%|*}; name=${spec##*|}
    for rep in 1 2; do
      GPUAR_LIBRARY=paper_1404_0027_b200/lib/exp_base.so timeout 300 python bench.py $args --no-cpu --no-e2e --no-it > $out/${name}_base_$rep.json 2>&1
      timeout 300 python bench.py $args --no-cpu --no-e2e --no-it > $out/${name}_new_$rep.json 2>&1
      echo "$name rep$rep base $(val $out/${name}_base_$rep.json) new $(val $out/${name}_new_$rep.json)"
    done
  done ;;
abn)
  out=gpurun_out/$1; libs=$2; shift 2; mkdir -p $out
  for spec in "$@"; do
    args=${spec%%|*}; name=${spec##*|}
    for rep in 1 2; do
      line="$name rep$rep"
      for lib in $libs; do
        if [ "$lib" = default ]; then L=paper_1404_0027_b200/lib/libgpuar.so; else L=paper_1404_0027_b200/lib/exp_$lib.so; fi
        GPUAR_LIBRARY=$L timeout 300 python bench.py $args --no-cpu --no-e2e --no-it > $out/${name}_${lib}_$rep.json 2>&1
        line="$line $lib $(val $out/${name}_${lib}_$rep.json)"
      done
      echo "$line"
    done
  done ;;
team-sweep)
  out=gpurun_out/${1:-team}; mkdir -p $out
  run() {
    name=$1; args=$2; shift 2; line="$name"
    for g in "$@"; do
      if [ $g = model ]; then env -u GPUAR_TEAM timeout 300 python bench.py $args --no-cpu --no-e2e > $out/${name}_$g.json 2>&1
      else GPUAR_TEAM=$g timeout 300 python bench.py $args --no-cpu --no-e2e > $out/${name}_$g.json 2>&1; fi
      line="$line | $g: $(val $out/${name}_$g.json)"
    done
    echo "$line"
  }
  run c2 "--config c2 --steps 300" model 8 16 32
  run c3p3 "--config c3 --dist pareto --M 1000 --steps 20" model 2 4 8 32
  run c3e3 "--config c3 --dist exponential --M 1000 --steps 20" model 1 2 4
  run c3u4 "--config c3 --dist uniform --M 10000 --steps 20" model 1 2
  run c1 "--config c1 --steps 300" model 1 2 4 ;;
divcheck)
  mkdir -p gpurun_out/div
  (cd scripts/ubench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o divcheck divcheck.cu) || exit 1
  timeout 1500 ./scripts/ubench/divcheck > gpurun_out/div/divcheck.txt 2>&1; echo "rc=$?" >> gpurun_out/div/divcheck.txt
  cat gpurun_out/div/divcheck.txt ;;
*)
  echo "unknown task $task"; exit 2 ;;
esac
