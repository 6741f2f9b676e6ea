# GPU-box session: ncu --set full (with source) of the fused BHHB kernel (cfg4).
mkdir -p gpurun_out
python tools/cfg.py cfg4 1 > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bhhb_fused -s 1 -c 1 -o gpurun_out/bf python tools/cfg.py cfg4 1 > /dev/null 2>&1
ncu -i gpurun_out/bf.ncu-rep --page raw --csv > gpurun_out/bf_raw.csv 2>/dev/null
ncu -i gpurun_out/bf.ncu-rep --page source --csv > gpurun_out/bf_source.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
