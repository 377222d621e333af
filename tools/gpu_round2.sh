# evidence refresh (session 2): per-config timings, gram captures
mkdir -p gpurun_out
timeout 1500 python tools/bench_configs.py --configs 1,2,3,4,5 --out gpurun_out/configs_r1s2.json > gpurun_out/configs.log 2>&1; echo configs rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:slab_gram_kernel -c 1 -o gpurun_out/slab_gram_full python tools/gram_bench.py --rows 16777216 --ncol 65 --reps 1 > gpurun_out/ncu_gram.log 2>&1; echo ncu_gram rc=$?
