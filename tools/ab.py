# Development helper: interleaved A/B timing of library env switches on one
# workload (python tools/ab.py cfg2 HK_PP_TWV=2 HK_PP_TWV=8 ...).  The library
# reads its HK_* switches at every launch, so one process serves all variants.
import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1401_6238_b200 import batched, workloads

which, variants = sys.argv[1], sys.argv[2:] or [""]
if which == "cfg2":
    h, x = workloads.cfg2()
    dh = torch.from_numpy(h).cuda(); dx = torch.from_numpy(x).cuda()
    y = torch.empty((4096, 1024), dtype=torch.complex128, device="cuda")
    f = lambda: batched.hankel_tvp_partial(dh, [dx, dx, dx], (1024,) * 4, out=y)
elif which == "cfg3":
    h, x = workloads.cfg3()
    dh = torch.from_numpy(h).cuda()[None]; dx = torch.from_numpy(x).cuda()[None]
    f = lambda: batched.hankel_tvp_partial(dh, [dx, dx], (1 << 22,) * 3)
elif which == "cfg4":
    Hb, X = workloads.cfg4()
    dH = torch.from_numpy(Hb).cuda()
    dxv = torch.from_numpy(np.ascontiguousarray(np.transpose(X, (0, 2, 1)))).cuda().reshape(1024, -1)
    f = lambda: batched.bhhb_tvp_partial(dH, [dxv, dxv], 3, (64,) * 3, (64,) * 3)
elif which == "cfg5":
    sig, U0, shape = workloads.cfg5(signals=256)
    dsig = torch.from_numpy(sig).cuda()
    dU = torch.from_numpy(np.ascontiguousarray(np.conj(U0))).cuda()[None].expand(256, -1, -1).contiguous()
    spec = batched.hankel_spectrum(dsig, shape)
    f = lambda: batched.times_matrices(spec, shape, [dU, dU], spectrum=True)

def setenv(v):
    for kv in v.split(","):
        if "=" in kv:
            k, val = kv.split("=", 1)
            os.environ[k] = val

def clear(v):
    for kv in v.split(","):
        if "=" in kv:
            os.environ.pop(kv.split("=", 1)[0], None)

reps, rounds = 20, 5
res = {v: [] for v in variants}
for r in range(rounds):
    for v in variants:
        setenv(v)
        for _ in range(3): f()
        torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps): f()
        e.record(); torch.cuda.synchronize()
        res[v].append(s.elapsed_time(e) / reps * 1e3)
        clear(v)
for v in variants:
    t = sorted(res[v])
    print(f"{which} [{v or 'default'}]: median {t[len(t)//2]:.1f} us  min {t[0]:.1f}  all {[round(x,1) for x in res[v]]}")
