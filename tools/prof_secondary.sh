# ncu --set full of the dominant kernels of cfg3/cfg4/cfg5, raw pages exported
# to gpurun_out/ (the .ncu-rep files are too large to bring back).  Each
# capture selects the kernel by name AND skips the warm-up launches of the
# same command (tools/cfg.py runs `reps` warm-up + `reps` timed calls), so
# the profiled launch is the steady-state one.
set -e
# cfg3: packed column pass (first k_cols launch of the 2nd call), 8192-point row stage
python tools/cfg.py cfg3 2 >/dev/null
ncu --set full --clock-control none -k regex:k_cols -s 2 -c 1 -o /tmp/p3c python tools/cfg.py cfg3 1 >/dev/null 2>&1
ncu -i /tmp/p3c.ncu-rep --page raw --csv > gpurun_out/p3_cols_raw.csv
ncu --set full --clock-control none -k regex:k_hankel_fast -s 1 -c 1 -o /tmp/p3r python tools/cfg.py cfg3 1 >/dev/null 2>&1
ncu -i /tmp/p3r.ncu-rep --page raw --csv > gpurun_out/p3_rows_raw.csv
# cfg3 final column pass (ST_C): the 2nd k_cols launch of a call (packed pass, rows, final)
ncu --set full --clock-control none -k regex:k_cols -s 3 -c 1 -o /tmp/p3f python tools/cfg.py cfg3 1 >/dev/null 2>&1
ncu -i /tmp/p3f.ncu-rep --page raw --csv > gpurun_out/p3_final_raw.csv
# cfg4 row stage
python tools/cfg.py cfg4 2 >/dev/null
ncu --set full --clock-control none -k regex:k_hankel_fast -s 1 -c 1 -o /tmp/p4r python tools/cfg.py cfg4 1 >/dev/null 2>&1
ncu -i /tmp/p4r.ncu-rep --page raw --csv > gpurun_out/p4_rows_raw.csv
# cfg5: the combo launch of times_matrices (k_hankel_fast with the spectrum
# inputs) -- per call: hk_spectrum is outside the timed loop, then one
# column-spectra launch and one combo launch, so skip 1 warm-up call (2
# launches) and the column-spectra launch of the second call
python tools/cfg.py cfg5 2 >/dev/null
ncu --set full --clock-control none -k regex:k_hankel_fast -s 4 -c 1 -o /tmp/p5 python tools/cfg.py cfg5 1 >/dev/null 2>&1
ncu -i /tmp/p5.ncu-rep --page raw --csv > gpurun_out/p5_combos_raw.csv
ncu -i /tmp/p5.ncu-rep --page details --csv | grep -m1 "Kernel Name\|k_hankel" > gpurun_out/p5_kernel_name.txt || true
echo done
