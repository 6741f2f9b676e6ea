# Development helper (run from the repo root: python tools/lat.py ...); not part of the package or the tests.
# Where does the numpy-facing latency of HankelTensor.tvp_partial go (cfg1)?
import sys, time, ctypes, numpy as np, torch
sys.path.insert(0, '.')
import paper_1401_6238_b200 as P
from paper_1401_6238_b200 import workloads, batched, _native as N, _device as D
h, x = workloads.cfg1()
H = P.HankelTensor((100,) * 3, h)
H.tvp_partial([x, x])
def t(fn, n=2000):
    for _ in range(50): fn()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    return (time.perf_counter() - t0) / n * 1e6
cache = H._dev if hasattr(H, "_dev") else None
print("full API            %.1f us" % t(lambda: H.tvp_partial([x, x])))
vecs = [H._pad(x, 1), H._pad(x, 2)]
print("_pad x2             %.1f us" % t(lambda: [H._pad(x, 1), H._pad(x, 2)]))
print("_partial (no pad)   %.1f us" % t(lambda: H._partial(vecs)))
print("_dedupe             %.1f us" % t(lambda: D._dedupe(vecs)))
print("hankel_plan         %.1f us" % t(lambda: batched.hankel_plan((100,) * 3, 0)))
print("current_stream      %.1f us" % t(lambda: torch.cuda.current_stream(0)))
print("cuda sync (idle)    %.1f us" % t(lambda: torch.cuda.synchronize()))
# raw C-ABI latency call (pinned zero-copy, kernel, stream sync) with prebuilt arguments
st = D._Staging.get(0)
plan, hop = H._dev._lean[0]
uniq, idx = D._dedupe(vecs)
n_in = sum(a.shape[0] for a in uniq)
st.ensure(n_in + 100)
xoff = (ctypes.c_int64 * len(idx))(*[0 for i in idx])
lib = N.load_library()
sp = ctypes.c_void_p(torch.cuda.current_stream(0).cuda_stream)
fn = lambda: lib.hk_tvp_partial_host(plan.handle, hop, st.hbase, n_in, xoff, len(idx), st.dbase,
                                     st.dbase + 16 * n_in, st.hbase + 16 * n_in, sp)
print("raw C call          %.1f us" % t(fn))
print("require_cuda        %.1f us" % t(lambda: D.require_cuda()))
print("_state              %.1f us" % t(lambda: H._dev._state()))
