# ncu --set full captures of the main non-fill kernels inside bench.py's timed region
# (one capture per kernel: S-hat GEMV, tile RK3 stage, seam filter, sampling/sets, eigen)
mkdir -p gpurun_out
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_k.json 2>&1; echo short rc=$?
for k in "gemv_gather_kernel<9, true, false>" stage_tile_kernel filter_kernel sets_kernel basis_kernel; do
  n=$(echo "$k" | cut -d'<' -f1)
  timeout 600 ncu --set full --clock-control none --nvtx --nvtx-include "timed/" -k regex:"$n" -c 1 -o gpurun_out/k_$n python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_$n.log 2>&1; echo "$n rc=$?"
done
