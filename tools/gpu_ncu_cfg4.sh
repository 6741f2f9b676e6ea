# GPU-box session: ncu --set full (with source) of the cfg4 kernels (tools/cfg.py cfg4 1 = two steps).
mkdir -p gpurun_out
python tools/cfg.py cfg4 1 > /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python tools/cfg.py cfg4 1 > /dev/null 2>&1
cap() {  # name, kernel regex, launches to skip
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o gpurun_out/$1 python tools/cfg.py cfg4 1 > /dev/null 2>&1
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  ncu -i gpurun_out/$1.ncu-rep --page source --csv > gpurun_out/$1_source.csv 2>/dev/null
  rm -f gpurun_out/$1.ncu-rep
}
cap c4_rows k_rows_pp 1
cap c4_col0 k_cols 3
cap c4_col1 k_cols 4
cap c4_col2 k_cols 5
