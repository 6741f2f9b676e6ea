# Development helper: aggregate ncu source-page (SASS) stall samples into the
# code segments between barriers (python tools/ncu_src_phases.py pp_source.csv).
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
cols = ["stall_barrier", "stall_long_sb", "stall_math", "stall_mio", "stall_not_selected",
        "stall_selected", "stall_short_sb", "stall_wait", "stall_no_inst", "stall_dispatch"]
seg, segs, tot = None, [], 0
def new(addr, src):
    return {"start": addr, "first": src, "n": 0, "samples": 0, **{c: 0 for c in cols}, "ops": {}}
seg = new("0", "entry")
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else ""
    if op.startswith("@"):
        op = src.split()[1]
    n = int(float(r[ix["# Samples"]] or 0))
    seg["samples"] += n; tot += n
    for c in cols:
        seg[c] += int(float(r[ix[c]] or 0))
    o = op.split(".")[0]
    seg["ops"][o] = seg["ops"].get(o, 0) + int(float(r[ix["Instructions Executed"]] or 0))
    if o in ("BAR", "WARPSYNC", "SYNCS") or "BAR" == o:
        segs.append(seg); seg = new(r[ix["Address"]], src)
segs.append(seg)
print("total samples", tot)
for s in segs:
    if s["samples"] < tot * 0.01:
        continue
    top = sorted(s["ops"].items(), key=lambda kv: -kv[1])[:6]
    st = ", ".join(f"{c[6:]}={s[c]}" for c in cols if s[c] > s["samples"] * 0.05)
    print(f"{s['start']:>6} {100*s['samples']/tot:5.1f}%  {st}\n        ops {top}\n        ends-after: {s['first'][:60]}")
