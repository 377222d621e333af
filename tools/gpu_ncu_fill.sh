# one ncu --set full capture of the dominant kernel (fill pass) inside bench.py's timed region
mkdir -p gpurun_out
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_short2.json 2>&1; echo short rc=$?
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" -k regex:fill_kernel -c 1 -o gpurun_out/fill_full python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_fill.log 2>&1; echo ncu rc=$?
