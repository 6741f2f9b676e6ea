# GPU-box session: parity tests of the ping-pong kernels, then interleaved A/B
# runs (tools/ab.py) of the variants named in AB2 / AB3 / AB4 on cfg2 / cfg3 / cfg4.
mkdir -p gpurun_out
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_r2_kernels.py tests/test_gpu_products.py tests/test_gpu_large.py} -m gpu -x -q > gpurun_out/ab_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab_test.log
[ -n "$AB2" ] && timeout 300 python tools/ab.py cfg2 $AB2 > gpurun_out/ab_cfg2.txt 2>&1
[ -n "$AB3" ] && timeout 300 python tools/ab.py cfg3 $AB3 > gpurun_out/ab_cfg3.txt 2>&1
[ -n "$AB4" ] && timeout 300 python tools/ab.py cfg4 $AB4 > gpurun_out/ab_cfg4.txt 2>&1
echo done > gpurun_out/ab_done
