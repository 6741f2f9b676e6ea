# Development helper (run from the repo root: python tools/configs.py ...); not part of the package or the tests.
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_1401_6238_b200 as P
from paper_1401_6238_b200 import batched, workloads

def dev_time(fn, reps=10, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps

# cfg1
h, x = workloads.cfg1()
dh = torch.from_numpy(h).cuda()[None]; dx = torch.from_numpy(x).cuda()[None]
ms = dev_time(lambda: batched.hankel_tvp_partial(dh, [dx, dx], (100,)*3), reps=200)
msf = dev_time(lambda: batched.hankel_tvp_full(dh, [dx, dx, dx], (100,)*3), reps=200)
H = P.HankelTensor((100,)*3, h); H.tvp_partial([x, x])
t0 = time.perf_counter(); [H.tvp_partial([x, x]) for _ in range(200)]; t1 = time.perf_counter()
print(f"cfg1: device partial {ms*1e3:.1f} us, full {msf*1e3:.1f} us; numpy API {1e6*(t1-t0)/200:.1f} us/call")
# cfg3
h, x = workloads.cfg3()
dh = torch.from_numpy(h).cuda()[None]; dx = torch.from_numpy(x).cuda()[None]
ms = dev_time(lambda: batched.hankel_tvp_partial(dh, [dx, dx], (1<<22,)*3), reps=5)
print(f"cfg3: {ms*1e3:.1f} us/product, B_alg 167.8 MB -> {167772144/(ms*1e-3)/1e9:.0f} GB/s")
# cfg4
Hb, X = workloads.cfg4()
dH = torch.from_numpy(Hb).cuda()
dxv = torch.from_numpy(np.ascontiguousarray(np.transpose(X, (0, 2, 1)))).cuda().reshape(1024, -1)
ms = dev_time(lambda: batched.bhhb_tvp_partial(dH, [dxv, dxv], 3, (64,)*3, (64,)*3), reps=5)
print(f"cfg4: {ms*1e3:.1f} us/batch, {1024/ms*1e3:.3e} products/s, {708672*1024/(ms*1e-3)/1e9:.0f} GB/s")
# cfg5 products
sig, U0, shape = workloads.cfg5(signals=256)
dsig = torch.from_numpy(sig).cuda()
dU = torch.from_numpy(np.ascontiguousarray(np.conj(U0))).cuda()[None].expand(256, -1, -1).contiguous()
spec = batched.hankel_spectrum(dsig, shape)
ms = dev_time(lambda: batched.times_matrices(spec, shape, [dU, dU], spectrum=True), reps=5)
print(f"cfg5: times_matrices 256 signals x 25 products: {ms*1e3:.1f} us -> {6400/ms*1e3:.3e} products/s")
