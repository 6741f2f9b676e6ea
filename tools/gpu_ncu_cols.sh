# GPU-box session: ncu --set full (with source) of the cfg3 packed column pass and final column pass.
# tools/cfg.py cfg3 1 runs two steps; k_cols launches in order: A, C, A, C.
mkdir -p gpurun_out
python tools/cfg.py cfg3 1 > /dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cols -s 2 -c 1 -o gpurun_out/cA python tools/cfg.py cfg3 1 > /dev/null 2>&1
ncu -i gpurun_out/cA.ncu-rep --page raw --csv > gpurun_out/cA_raw.csv 2>/dev/null
ncu -i gpurun_out/cA.ncu-rep --page source --csv > gpurun_out/cA_source.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cols -s 3 -c 1 -o gpurun_out/cC python tools/cfg.py cfg3 1 > /dev/null 2>&1
ncu -i gpurun_out/cC.ncu-rep --page raw --csv > gpurun_out/cC_raw.csv 2>/dev/null
ncu -i gpurun_out/cC.ncu-rep --page source --csv > gpurun_out/cC_source.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
