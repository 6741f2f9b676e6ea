# Development helper (run from the repo root: python tools/cfg.py ...); not part of the package or the tests.
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1401_6238_b200 import batched, workloads
which = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if which == "cfg1":
    h, x = workloads.cfg1()
    dh = torch.from_numpy(h).cuda()[None]; dx = torch.from_numpy(x).cuda()[None]
    f = lambda: batched.hankel_tvp_partial(dh, [dx, dx], (100,)*3)
elif which == "cfg2":
    h, x = workloads.cfg2()
    dh = torch.from_numpy(h).cuda(); dx = torch.from_numpy(x).cuda()
    y = torch.empty((4096, 1024), dtype=torch.complex128, device="cuda")
    f = lambda: batched.hankel_tvp_partial(dh, [dx, dx, dx], (1024,)*4, out=y)
elif which == "cfg4":
    Hb, X = workloads.cfg4()
    dH = torch.from_numpy(Hb).cuda()
    dxv = torch.from_numpy(np.ascontiguousarray(np.transpose(X, (0, 2, 1)))).cuda().reshape(1024, -1)
    f = lambda: batched.bhhb_tvp_partial(dH, [dxv, dxv], 3, (64,)*3, (64,)*3)
elif which == "cfg3":
    h, x = workloads.cfg3()
    dh = torch.from_numpy(h).cuda()[None]; dx = torch.from_numpy(x).cuda()[None]
    f = lambda: batched.hankel_tvp_partial(dh, [dx, dx], (1 << 22,)*3)
elif which == "cfg5":
    sig, U0, shape = workloads.cfg5(signals=256)
    dsig = torch.from_numpy(sig).cuda()
    dU = torch.from_numpy(np.ascontiguousarray(np.conj(U0))).cuda()[None].expand(256, -1, -1).contiguous()
    spec = batched.hankel_spectrum(dsig, shape)
    f = lambda: batched.times_matrices(spec, shape, [dU, dU], spectrum=True)
for _ in range(reps): f()
torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(reps): f()
e.record(); torch.cuda.synchronize()
print(f"{which}: {s.elapsed_time(e) / reps * 1e3:.1f} us/step")
