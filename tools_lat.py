import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_1401_6238_b200 as P
from paper_1401_6238_b200 import workloads
h, x = workloads.cfg1()
H = P.HankelTensor((100,)*3, h)
for _ in range(20): H.tvp_partial([x, x])
import cProfile, pstats
t0 = time.perf_counter()
for _ in range(500): H.tvp_partial([x, x])
print("us/call", (time.perf_counter() - t0) / 500 * 1e6)
cProfile.run("for _ in range(200): H.tvp_partial([x, x])", "/tmp/prof.out")
pstats.Stats("/tmp/prof.out").sort_stats("tottime").print_stats(12)
