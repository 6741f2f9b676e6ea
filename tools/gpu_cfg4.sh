# GPU-box session: two-level parity tests (1D four-step and 2D block), then cfg4 / cfg3 timing.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_large.py tests/test_gpu_r2_kernels.py tests/test_gpu_r2_parity.py tests/test_gpu_fuzz.py tests/test_gpu_products.py -m gpu -x -q > gpurun_out/gputest_cfg4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_cfg4.log
tail -4 gpurun_out/gputest_cfg4.log
timeout 300 python tools/ab.py cfg4 ${AB_VARIANTS:-""} 2>&1 | tee gpurun_out/ab_cfg4.txt
timeout 300 python tools/ab.py cfg3 "" HK_NO_COLTMA=1 2>&1 | tee -a gpurun_out/ab_cfg4.txt
