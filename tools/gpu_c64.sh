# GPU-box session: complex64 parity tests, then cfg2-c64 timing of the ping-pong kernel variants.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_c64.py -m gpu -x -q > gpurun_out/gputest_c64.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_c64.log
HK_PP_C64_NG=3 timeout 900 python -m pytest tests/test_gpu_c64.py -m gpu -x -q >> gpurun_out/gputest_c64.log 2>&1; echo "pytest NG=3 rc=$?" >> gpurun_out/gputest_c64.log
tail -6 gpurun_out/gputest_c64.log
timeout 200 python tools/c64.py 2>&1 | tee gpurun_out/c64_time.txt
HK_PP_C64_NG=3 timeout 200 python tools/c64.py 2>&1 | tee -a gpurun_out/c64_time.txt
HK_NO_PP_C64=1 timeout 200 python tools/c64.py 2>&1 | tee -a gpurun_out/c64_time.txt
