# GPU-box session: all GPU tests then the default bench line (both arms).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/c_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c_gputest.log
timeout 900 python bench.py > gpurun_out/c_bench.json 2> gpurun_out/c_bench.err; echo "bench rc=$?" >> gpurun_out/c_bench.err
tail -3 gpurun_out/c_gputest.log; cat gpurun_out/c_bench.json | cut -c1-1500
