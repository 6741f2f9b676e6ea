# GPU-box session: all GPU tests, then interleaved timing of every config.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/c_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c_gputest.log
tail -3 gpurun_out/c_gputest.log
for c in cfg5 cfg4 cfg3 cfg2; do timeout 300 python tools/ab.py $c "" 2>&1 | tail -1; done | tee gpurun_out/c_times.txt
