# GPU-box session: cfg3 A/B of column-tile widths + per-kernel launch list.
mkdir -p gpurun_out
timeout 300 python tools/ab.py cfg3 ${AB3:-HK_COL1536_TILE=4 HK_COL1536_TILE=2 HK_COL1536_TILE=1} > gpurun_out/ab3.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 12 --csv --log-file gpurun_out/l3.csv python tools/cfg.py cfg3 2 > /dev/null 2>&1
