# GPU-box session: parity tests of the 1D products, then an interleaved A/B on cfg2.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_products.py tests/test_gpu_fuzz.py tests/test_gpu_determinism.py -m gpu -x -q > gpurun_out/gputest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_quick.log
timeout 300 python tools/ab.py cfg2 ${AB_VARIANTS:-HK_PP_TWV=2 HK_PP_TWV=8} > gpurun_out/ab.txt 2>&1
