# Development helper: static SASS opcode counts per kernel of an object file
# (python tools/sass_count.py build/obj/hk_pp1d.o [name-filter]).
import re, subprocess, sys
sass = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
filt = sys.argv[2] if len(sys.argv) > 2 else ""
cur, cnt = None, {}
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1); cnt[cur] = {}; continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
    if m and cur:
        op = m.group(2)
        cnt[cur][op] = cnt[cur].get(op, 0) + 1
keys = ["DADD", "DFMA", "DMUL", "LDS", "STS", "LDTM", "STTM", "BAR", "LDG", "STG"]
for f, c in cnt.items():
    if filt in f:
        fp = c.get("DADD", 0) + c.get("DFMA", 0) + c.get("DMUL", 0)
        print(f[-40:], {k: c.get(k, 0) for k in keys}, "fp64", fp, "total", sum(c.values()))
