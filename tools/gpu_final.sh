# round evidence (session 2): gpu tests, default bench line, launch list of the timed region,
# ncu --set full captures of the fill kernel and of the main non-fill kernels (each ncu only after
# its command exited 0 without ncu)
mkdir -p gpurun_out
bash tools/gpu_round.sh
bash tools/gpu_ncu_kernels.sh
