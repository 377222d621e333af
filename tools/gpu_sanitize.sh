#!/bin/bash
# compute-sanitizer evidence (cooperative grid barriers, speculative filter passes,
# mbarrier pipelines): memcheck, racecheck (shared-memory hazards), synccheck (barrier misuse),
# initcheck on configs 1 and 2 through tools/sanitize_run.py.  Logs -> gpurun_out/, summarised
# into profiles/ by the caller.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for c in 1 2; do
  for tool in memcheck racecheck synccheck initcheck; do
    extra=""
    [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
    timeout 1500 $CS --tool $tool $extra --print-limit 50 --log-file gpurun_out/san_${tool}_c${c}.log \
      python tools/sanitize_run.py $c 2 > gpurun_out/san_${tool}_c${c}.out 2>&1
    echo "config $c $tool rc=$? $(tail -1 gpurun_out/san_${tool}_c${c}.log)"
  done
done
