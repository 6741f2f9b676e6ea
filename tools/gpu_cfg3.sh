# GPU-box session: two-level parity tests, then cfg3 A/B of the column-kernel switches.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_r2_kernels.py tests/test_gpu_r2_parity.py -m gpu -x -q > gpurun_out/gputest_cfg3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_cfg3.log
tail -4 gpurun_out/gputest_cfg3.log
timeout 300 python tools/ab.py cfg3 ${AB_VARIANTS:-""} 2>&1 | tee gpurun_out/ab_cfg3.txt
