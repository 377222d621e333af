# round-end evidence: gpu tests, default bench line, launch list of the timed region, one
# ncu --set full capture of the fill kernel (each ncu only after its command exited 0 without ncu)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_short.json 2>&1; echo short rc=$?
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo ncu rc=$?
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" -k regex:fill_kernel -c 1 -o gpurun_out/fill_full python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_fill.log 2>&1; echo ncu_full rc=$?
