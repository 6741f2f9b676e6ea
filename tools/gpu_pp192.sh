# GPU-box session: 192-point ping-pong row kernel (HK_PP192=1): block parity tests, then cfg4 timing with and without.
mkdir -p gpurun_out
HK_PP192=1 timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_fuzz.py tests/test_gpu_r2_kernels.py -m gpu -x -q -k "block or cfg4 or bhhb or BHHB" > gpurun_out/gputest_pp192.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_pp192.log
tail -4 gpurun_out/gputest_pp192.log
HK_PP192=1 timeout 300 python tools/ab.py cfg4 "" 2>&1 | tee gpurun_out/ab_pp192.txt
timeout 300 python tools/ab.py cfg4 "" 2>&1 | tee -a gpurun_out/ab_pp192.txt
