# Development helper (run from the repo root: python tools/ncu_summary.py ...); not part of the package or the tests.
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
keys = sys.argv[2:] or ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
  "launch__registers_per_thread", "launch__occupancy_limit", "sm__warps_active.avg.pct_of_peak_sustained_active",
  "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
  "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
  "smsp__average_warp", "smsp__warp_issue_stalled", "sass__inst_executed_register_spilling", "smsp__inst_executed.sum",
  "sm__inst_executed_pipe_lsu", "l1tex__data_pipe_lsu_wavefronts.sum", "lts__t_bytes.sum", "dram__throughput.avg.pct"]
for i, h in enumerate(hdr):
    if any(k in h for k in keys) and "pct_of_peak_sustained_elapsed" not in h.replace("dram__throughput.avg.pct_of_peak_sustained_elapsed","KEEP"):
        print(f"{h:90s} {vals[i]:>20s} {units[i]}")
