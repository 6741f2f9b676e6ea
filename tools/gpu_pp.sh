# GPU-box session: GPU tests, cfg2 twiddle-source A/B, bench, ncu of the pp kernel.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 300 python tools/ab.py cfg2 HK_PP_TWV=2 HK_PP_TWV=8 HK_NO_PP=1 > gpurun_out/ab.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hankel_pp -s 2 -c 1 -o gpurun_out/pp python tools/cfg.py cfg2 2 > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/pp.ncu-rep --page raw --csv > gpurun_out/pp_raw.csv 2>/dev/null
ncu -i gpurun_out/pp.ncu-rep --page source --csv > gpurun_out/pp_source.csv 2>/dev/null
rm -f gpurun_out/pp.ncu-rep
