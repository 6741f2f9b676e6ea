# GPU-box session (round 2, re-entry checkpoint): every GPU test, the default
# bench line, then compute-sanitizer memcheck/racecheck/synccheck over every
# kernel variant (tools/sanitize.py), each bounded by its own timeout.
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/s_env.txt 2>&1
which compute-sanitizer >> gpurun_out/s_env.txt 2>&1
compute-sanitizer --version >> gpurun_out/s_env.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s_gputest.log
timeout 900 python bench.py > gpurun_out/s_bench.json 2> gpurun_out/s_bench.err; echo "bench rc=$?" >> gpurun_out/s_bench.err
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize.py > gpurun_out/s_san_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/s_san_$tool.log
done
echo done > gpurun_out/s_done
