#!/bin/bash
# ncu --set full captures (one launch each) of the round-2 kernels inside bench.py's timed region
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_k2.json 2>&1; echo short rc=$?
for k in ${KERNELS:-fill_kernel gather_gram_kernel gemv_gather_kernel solve_kernel refine_kernel basis_kernel}; do
  timeout 600 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" -k regex:"$k" -c 1 \
    -o gpurun_out/r2_$k python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_r2_$k.log 2>&1
  echo "$k rc=$?"
  python tools/ncu_summary.py gpurun_out/r2_$k.ncu-rep > gpurun_out/r2_$k.txt 2>&1
done
