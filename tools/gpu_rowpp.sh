# GPU-box session: cfg2/cfg3 timings + ncu (with source) of the cfg3 row-stage ping-pong kernel.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_large.py tests/test_gpu_products.py -m gpu -x -q > gpurun_out/gt_q.log 2>&1
timeout 300 python tools/ab.py cfg2 "" > gpurun_out/ab.txt 2>&1
timeout 300 python tools/ab.py cfg3 "" HK_NO_PP_ROWS=1 >> gpurun_out/ab.txt 2>&1
python tools/cfg.py cfg3 1 > /dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hankel_pp -s 1 -c 1 -o gpurun_out/rp python tools/cfg.py cfg3 1 > /dev/null 2>&1
ncu -i gpurun_out/rp.ncu-rep --page raw --csv > gpurun_out/rp_raw.csv 2>/dev/null
ncu -i gpurun_out/rp.ncu-rep --page source --csv > gpurun_out/rp_source.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
