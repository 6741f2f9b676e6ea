# GPU-box session: ncu --set full of one steady-state cfg2 ping-pong launch, raw + source pages.
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hankel_pp -s 2 -c 1 -o gpurun_out/pp python tools/cfg.py cfg2 2 > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/pp.ncu-rep --page raw --csv > gpurun_out/pp_raw.csv 2>/dev/null
ncu -i gpurun_out/pp.ncu-rep --page source --csv > gpurun_out/pp_source.csv 2>/dev/null
ncu -i gpurun_out/pp.ncu-rep --page details --csv > gpurun_out/pp_details.csv 2>/dev/null
rm -f gpurun_out/pp.ncu-rep
