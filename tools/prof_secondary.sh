# ncu --set full of the dominant kernels of cfg3/cfg4/cfg5, raw pages exported
# to gpurun_out/ (the .ncu-rep files are too large to bring back).
set -e
python tools/cfg.py cfg3 2 >/dev/null
ncu --set full --clock-control none -k regex:k_cols -s 0 -c 1 -o /tmp/p3c python tools/cfg.py cfg3 1 >/dev/null 2>&1
ncu -i /tmp/p3c.ncu-rep --page raw --csv > gpurun_out/p3_cols_raw.csv
ncu --set full --clock-control none -k regex:k_hankel_fast -s 0 -c 1 -o /tmp/p3r python tools/cfg.py cfg3 1 >/dev/null 2>&1
ncu -i /tmp/p3r.ncu-rep --page raw --csv > gpurun_out/p3_rows_raw.csv
python tools/cfg.py cfg4 2 >/dev/null
ncu --set full --clock-control none -k regex:k_hankel_fast -s 0 -c 1 -o /tmp/p4r python tools/cfg.py cfg4 1 >/dev/null 2>&1
ncu -i /tmp/p4r.ncu-rep --page raw --csv > gpurun_out/p4_rows_raw.csv
python tools/cfg.py cfg5 2 >/dev/null
ncu --set full --clock-control none -k regex:k_hankel_fast -s 1 -c 1 -o /tmp/p5 python tools/cfg.py cfg5 1 >/dev/null 2>&1
ncu -i /tmp/p5.ncu-rep --page raw --csv > gpurun_out/p5_combos_raw.csv
echo done
