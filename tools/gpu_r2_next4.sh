#!/bin/bash
# NEXT-4 GPU evidence: the implicit-HDM parity tests, the spectral-gap probe of the bench
# workload, and compute-sanitizer runs (memcheck / racecheck / synccheck) of configs 1-2.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_implicit.py -v -p no:cacheprovider > gpurun_out/pytest_implicit.txt 2>&1
echo "implicit tests rc=$? $(tail -1 gpurun_out/pytest_implicit.txt)"
timeout 300 python tools/gap_probe.py 4 30 > gpurun_out/gap_probe_c4.json 2> gpurun_out/gap_probe_c4.err
echo "gap probe rc=$?"
CS=/usr/local/cuda/bin/compute-sanitizer
for c in 1 sod; do
  for tool in memcheck racecheck synccheck; do
    extra=""
    [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
    timeout 900 $CS --tool $tool $extra --print-limit 50 --log-file gpurun_out/san_${tool}_c${c}.log \
      python tools/sanitize_run.py $c 2 > gpurun_out/san_${tool}_c${c}.out 2>&1
    echo "config $c $tool rc=$? $(tail -1 gpurun_out/san_${tool}_c${c}.log)"
  done
done
