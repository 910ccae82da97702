# round-2 ncu captures of the kernels the round changed (one report each, launch-skipped past warm-up)
bash scripts/probes/ncu_kernel.sh r2_pipe_efsignsgd k_bucket_pipe --codec efsignsgd
bash scripts/probes/ncu_kernel.sh r2_rng_emit_qsgd k_rng_emit --codec qsgd
bash scripts/probes/ncu_kernel.sh r2_randk_tables k_randk_tables --codec randk --sparsity 0.99
ncu --set full --clock-control none --import-source on -k regex:k_randk_emit\< -c 1 -f -o gpurun_out/r2_randk_emit python bench.py --steps 1 --warmup 1 --no-search --no-cpu-baseline --e2e-steps 1 --codec randk --sparsity 0.99 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_decode -s 2 -c 1 -f -o gpurun_out/r2_decode_tab8 python scripts/probes/decode_nranks.py efsignsgd 8 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_decode -s 2 -c 1 -f -o gpurun_out/r2_decode_int8_8 python scripts/probes/decode_nranks.py int8 8 > /dev/null 2>&1
ls -la gpurun_out/r2_*.ncu-rep
