# GPU-box session: times_matrices / HOOI parity tests, then cfg5 A/B of the premultiplied spectra.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_hooi.py tests/test_gpu_r2_parity.py tests/test_gpu_fuzz.py tests/test_gpu_products.py tests/test_capi.py tests/test_gpu_determinism.py -m gpu -x -q > gpurun_out/gputest_cfg5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_cfg5.log
tail -4 gpurun_out/gputest_cfg5.log
timeout 300 python tools/ab.py cfg5 "" HK_NO_PREMUL=1 2>&1 | tee gpurun_out/ab_cfg5.txt
