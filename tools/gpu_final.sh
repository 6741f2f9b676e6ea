# GPU-box session (round-end evidence): all GPU tests, the default bench line,
# the ncu launch list of the same bench, and ncu --set full raw pages of the
# dominant kernel of every config.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f_gputest.log
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "bench rc=$?" >> gpurun_out/f_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
cap() {  # name, kernel regex, launches to skip, cfg
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o gpurun_out/f_$1 python tools/cfg.py $4 > /dev/null 2>&1
  ncu -i gpurun_out/f_$1.ncu-rep --page raw --csv > gpurun_out/f_$1_raw.csv 2>/dev/null
  ncu -i gpurun_out/f_$1.ncu-rep --page source --csv > gpurun_out/f_$1_source.csv 2>/dev/null
  rm -f gpurun_out/f_$1.ncu-rep
}
cap cfg2_pp k_hankel_pp 2 "cfg2 2"
cap cfg3_colA k_cols_tma 2 "cfg3 1"
cap cfg3_rows k_hankel_pp 1 "cfg3 1"
cap cfg3_colC k_cols_tma 3 "cfg3 1"
cap cfg4_rows k_rows_pp 1 "cfg4 1"
cap cfg4_hcols k_cols 3 "cfg4 1"
cap cfg4_xcols k_cols 4 "cfg4 1"
cap cfg4_ycols k_cols 5 "cfg4 1"
cap cfg5_combo k_hankel_fast 4 "cfg5 1"
python tools/raw_summary.py "cfg2 headline=gpurun_out/f_cfg2_pp_raw.csv" "cfg3 packed column pass=gpurun_out/f_cfg3_colA_raw.csv" \
  "cfg3 row stage=gpurun_out/f_cfg3_rows_raw.csv" "cfg3 final column pass=gpurun_out/f_cfg3_colC_raw.csv" \
  "cfg4 h column pass=gpurun_out/f_cfg4_hcols_raw.csv" "cfg4 x column pass=gpurun_out/f_cfg4_xcols_raw.csv" \
  "cfg4 row stage=gpurun_out/f_cfg4_rows_raw.csv" "cfg4 final column pass=gpurun_out/f_cfg4_ycols_raw.csv" \
  "cfg5 combo products=gpurun_out/f_cfg5_combo_raw.csv" > gpurun_out/f_summary.txt
echo done > gpurun_out/f_done
