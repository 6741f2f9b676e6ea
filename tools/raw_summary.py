# Development helper: one-paragraph summary of ncu raw-page CSVs
# (python tools/raw_summary.py "label=path_raw.csv" ...), the format of profiles/*_summary.txt.
import csv, sys
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"]
for arg in sys.argv[1:]:
    label, path = arg.split("=", 1)
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        print(f"== {label}: no capture"); continue
    hdr, units, vals = rows[0], rows[1], rows[2]
    ix = {h: i for i, h in enumerate(hdr)}
    print(f"== {label}: {vals[ix['Kernel Name']]}")
    for k in KEYS:
        if k in ix:
            print(f"   {k:82s} {vals[ix[k]]:>16s} {units[ix[k]]}")
    st = []
    for h, i in ix.items():
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                v = float(vals[i])
            except ValueError:
                continue
            if v > 0.3:
                st.append((v, h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
    print("   stalls/issue: " + ", ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)))
