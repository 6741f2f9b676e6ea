# GPU-box session: ncu --set full of one steady-state launch of the complex64 ping-pong kernel (cfg2-c64).
mkdir -p gpurun_out
python tools/c64.py > gpurun_out/c64_time.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hankel_pp_c64 -s 2 -c 1 -o gpurun_out/c64pp python tools/c64.py > /dev/null 2>&1
ncu -i gpurun_out/c64pp.ncu-rep --page raw --csv > gpurun_out/c64pp_raw.csv 2>/dev/null
rm -f gpurun_out/c64pp.ncu-rep
python tools/raw_summary.py "cfg2-c64 ping-pong kernel=gpurun_out/c64pp_raw.csv" > gpurun_out/c64pp_summary.txt
python - <<'PY' >> gpurun_out/c64pp_summary.txt
import csv
rows = list(csv.reader(open('gpurun_out/c64pp_raw.csv')))
h, u, v = rows[0], rows[1], rows[2]
for i, k in enumerate(h):
    if k in ('sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', 'sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active',
             'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active', 'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active'):
        print(f"   {k:82s} {v[i]:>16s} {u[i]}")
PY
