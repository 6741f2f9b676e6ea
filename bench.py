"""Benchmark: batched Hankel H·x^{m-1} products/s and % of HBM roofline.

Workload (BASELINE.json configs[1], "cfg2"): 4096 independent order-4,
n=1024 complex128 Hankel tensors, one x each, y_b = H_b x_b^3 with the FFT
length padded to 4096.  One step = one pass of the fused product over the
whole batch.  Inputs are seeded synthetic data of the stated shapes and
distributions (paper_1401_6238_b200.workloads.cfg2); they total 335 MB + 67 MB
of output per step, larger than the 126 MB L2, so no flush is needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU: one process per GPU.  ``--gpus N`` outside torchrun
re-launches itself under ``torch.distributed.run`` (127.0.0.1).  The 4096
products are sharded contiguously over the ranks (``dist.shard_range``; no
collective on the data path) -- strong scaling, the headline ``value``; each
rank then also runs a full 4096-product batch (weak scaling, ``weak``).
The result gather to rank 0 (NCCL gather) is timed separately (``gather``).
Every time is taken on the device with CUDA events and is the max over ranks.

The timed region replays the K steps from one CUDA graph (the product kernel
launched K times back to back, no host launch overhead between steps); the
per-launch kernel time of the roofline is measured with events around each
launch in a separate loop.

--impl reference times the reference's own CPU path on all host cores, rank 0
only (oracle/cpu_baseline.py): the unmodified reference package installed in
baseline/_ref when present (kind "reference"), else the pinned numpy port
(kind "port").  ``value`` is the reference's faster pow2 variant of the same
product (cli.py:277-291, L = 4096 like ours); the exact-length public API
(hankel.py:140-147, L = d_H = 4093) is reported beside it.
"""

from __future__ import annotations

import argparse
import importlib
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_MODE, ORDER, FFT_LEN = 1024, 4, 4096
# HK_BENCH_BATCH shrinks the batch for the CPU (gloo) harness test only
BATCH = int(os.environ.get("HK_BENCH_BATCH", "4096"))
DOF = ORDER * (N_MODE - 1) + 1
B_ALG = (DOF + N_MODE + N_MODE) * 16          # compulsory bytes per product
METRIC = "Hankel T·x^{m-1} products/s and % of HBM roofline at 1/2/4/8 B200"
UNIT = "products/s"
WORKLOAD = ("cfg2: 4096 independent order-4 n=1024 complex128 Hankel tensors, "
            "y_b = H_b x_b^3, FFT length 4096")


def peaks():
    out = {"hbm_gbs": 6650.0, "hbm_kind": "fallback (B200_PROFILING.md)", "fp64_tflops": None}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        out["hbm_gbs"], out["hbm_kind"] = float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        pass
    try:
        with open(os.path.join(ROOT, "profiles", "r02_ubench_fp64.json")) as f:
            r = json.load(f)["results"]
        out["fp64_tflops"] = next(x["dfma_tflops"] for x in r if x["mode"] == "DFMA only")
    except Exception:
        pass
    return out


def ncu_summary():
    """Per-launch DRAM bytes and FP64 pipe share of the dominant kernel from the
    committed ncu capture (profiles/ncu_summary.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


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
                 "-i", str(self.gpu), "-lms", "20"],
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


# ---------------------------------------------------------------- engines
class EventTimer:
    """CUDA events on the current stream, synchronised on read."""

    def __init__(self, torch):
        self.torch = torch
        self.a = torch.cuda.Event(enable_timing=True)
        self.b = torch.cuda.Event(enable_timing=True)

    def start(self):
        self.a.record()

    def stop(self):
        self.b.record()

    def ms(self):
        self.torch.cuda.synchronize()
        return self.a.elapsed_time(self.b)


class CudaEngine:
    """The product path under test: batched.hankel_tvp_partial on this rank's GPU
    (one fused kernel launch per step over the rank's products)."""

    backend = "nccl"
    launches_per_step = 1
    dtype = "c128"

    def __init__(self, local_rank):
        import torch

        self.torch = torch
        torch.cuda.set_device(local_rank)
        self.dev = torch.cuda.current_device()
        self.shape = (N_MODE,) * ORDER
        self._h = self._x = None

    def device(self):
        return self.torch.device("cuda", self.dev)

    def gpu_index(self):
        return self.dev

    def inputs(self):
        from paper_1401_6238_b200 import workloads

        if self._h is None:
            h, x = workloads.cfg2(4096, N_MODE, ORDER)  # BATCH < 4096: a prefix
            self._h, self._x = h[:BATCH], x[:BATCH]
        return self._h, self._x

    def load(self, lo, hi):
        torch = self.torch
        h, x = self.inputs()
        self.lo, self.hi = lo, hi
        self.dh = torch.from_numpy(h[lo:hi]).to(self.dev)
        self.dx = torch.from_numpy(x[lo:hi]).to(self.dev)
        self.y = torch.empty((hi - lo, N_MODE), dtype=torch.complex128, device=self.dev)

    def unload(self):
        self.dh = self.dx = self.y = None
        self.torch.cuda.empty_cache()

    def step(self):
        from paper_1401_6238_b200 import batched

        if self.hi > self.lo:
            batched.hankel_tvp_partial(self.dh, [self.dx, self.dx, self.dx], self.shape,
                                       out=self.y)

    def sync(self):
        self.torch.cuda.synchronize()

    def timer(self):
        return EventTimer(self.torch)

    def capture(self, k):
        """k steps in one CUDA graph; returns the replay callable."""
        torch = self.torch
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self.step()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(k):
                self.step()
        self._graph = g
        return g.replay

    def result(self):
        return self.y

    def e2e(self, steps, barrier, reduce_max):
        """The same products through the public host API: pinned host inputs ->
        H2D -> kernel -> D2H into pinned host memory, every step."""
        torch = self.torch
        from paper_1401_6238_b200 import batched

        h, x = self.inputs()
        lo, hi = self.lo, self.hi
        hp = torch.from_numpy(h[lo:hi]).pin_memory()
        xp = torch.from_numpy(x[lo:hi]).pin_memory()
        yp = torch.empty((hi - lo, N_MODE), dtype=torch.complex128, pin_memory=True)
        run = lambda: batched.hankel_tvp_partial_host(hp, [xp, xp, xp], self.shape, out=yp)
        for _ in range(2):
            run()
        torch.cuda.synchronize()
        barrier()
        t = self.timer()
        t.start()
        for _ in range(steps):
            run()
        t.stop()
        ms = reduce_max(t.ms())
        return ms, int(hp.numel() * 16 + xp.numel() * 16), int(yp.numel() * 16)


def load_engine(spec, local_rank):
    if not spec:
        return CudaEngine(local_rank)
    mod, _, cls = spec.partition(":")
    return getattr(importlib.import_module(mod), cls)(local_rank)


def parity_vs_golden(y, batch):
    """Relative error of this run's outputs against the reference's own cfg2
    outputs (tests/golden/cfg2.npz: products 0,1,2,4095 in full, the norm and
    first entry of every product)."""
    g = np.load(os.path.join(ROOT, "tests", "golden", "cfg2.npz"))
    sel = [int(s) for s in g["sel"] if s < batch]
    errs = [float(np.linalg.norm(y[s] - g["y"][k]) / np.linalg.norm(g["y"][k]))
            for k, s in enumerate(g["sel"]) if s < batch]
    norms = np.linalg.norm(y, axis=1)
    norm_err = float(np.max(np.abs(norms - g["norms"][:batch]) / g["norms"][:batch]))
    first_err = float(np.max(np.abs(y[:, 0] - g["first"][:batch]) / g["norms"][:batch]))
    return {"parity_rel_err": max(errs + [norm_err, first_err]),
            "parity_products_full": sel, "parity_norms_checked": int(batch),
            "parity_reference": "tests/golden/cfg2.npz (reference hankel.py:140-147 output)"}


# ---------------------------------------------------------------- harness
def measure(engine, steps, warmup, rank, world, barrier, reduce_max, weak=True, e2e=True):
    """Strong-scaling timed region over this rank's shard, per-launch kernel
    times, the timed gather, and (world > 1) the weak-scaling batch."""
    from paper_1401_6238_b200.dist import gather_shards, shard_range

    lo, hi = shard_range(BATCH, rank, world)
    engine.load(lo, hi)
    for _ in range(max(3, warmup)):
        engine.step()
    engine.sync()
    replay = engine.capture(steps) if hasattr(engine, "capture") else None
    clocks = ClockSampler(engine.gpu_index()) if hasattr(engine, "gpu_index") else None
    if clocks:
        clocks.start()
        time.sleep(0.25)
    out = {"shard": [lo, hi]}
    # -- strong scaling: the 4096-product batch sharded over the ranks
    barrier()
    engine.sync()
    t = engine.timer()
    t.start()
    if replay is not None:
        replay()
    else:
        for _ in range(steps):
            engine.step()
    t.stop()
    ms = t.ms()
    barrier()
    # -- per-launch kernel time (events around every launch, same stream)
    ev = []
    for _ in range(steps):
        tk = engine.timer()
        tk.start()
        engine.step()
        tk.stop()
        ev.append(tk)
    kern = statistics.mean(tk.ms() for tk in ev)
    out["clocks"] = clocks.stop() if clocks else None
    out["ms_total"] = reduce_max(ms)
    out["kernel_ms"] = reduce_max(kern)
    # -- result gather to rank 0, timed on its own
    barrier()
    engine.sync()
    tg = engine.timer()
    tg.start()
    full = gather_shards(engine.result(), BATCH, dst=0)
    tg.stop()
    out["gather_ms"] = reduce_max(tg.ms())
    out["full"] = None if full is None else full.cpu().numpy()
    # -- end to end through the public host API
    if e2e:
        out["e2e_ms"], out["h2d"], out["d2h"] = engine.e2e(steps, barrier, reduce_max)
    # -- weak scaling: every rank runs a full batch
    if weak and world > 1:
        engine.unload()
        engine.load(0, BATCH)
        for _ in range(3):
            engine.step()
        engine.sync()
        replay = engine.capture(steps) if hasattr(engine, "capture") else None
        barrier()
        engine.sync()
        t = engine.timer()
        t.start()
        if replay is not None:
            replay()
        else:
            for _ in range(steps):
                engine.step()
        t.stop()
        out["weak_ms_total"] = reduce_max(t.ms())
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1401_6238_b200.dist import max_over_ranks

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    engine = load_engine(args.engine, local)
    if world > 1:
        if engine.backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=engine.device())
        else:
            dist.init_process_group(engine.backend)
    coll_dev = engine.device()

    def barrier():
        if world > 1:
            dist.barrier()

    reduce_max = lambda v: max_over_ranks(v, coll_dev)
    r = measure(engine, args.steps, args.warmup, rank, world, barrier, reduce_max,
                e2e=not args.no_e2e)
    ms_step = r["ms_total"] / args.steps
    value = BATCH * args.steps / (r["ms_total"] * 1e-3)
    if rank == 0:
        pk = peaks()
        ncu = ncu_summary()
        # per-launch algorithmic bytes of the dominant kernel: rank 0's shard
        shard = r["shard"][1] - r["shard"][0]
        achieved = B_ALG * shard / (r["kernel_ms"] * 1e-3) / 1e9
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": engine.dtype,
            "data": "synthetic (seeded N(0,1) complex, SURVEY §8d cfg2)",
            "config": {"workload": WORKLOAD, "batch": BATCH, "products_per_gpu": shard,
                       "n": N_MODE, "order": ORDER, "fft_len": FFT_LEN,
                       "parallelism": f"dp{world} (batch sharded, no data-path collective)",
                       "l2": "inputs larger than L2 (402 MB/step vs 126 MB); no flush",
                       "timed_region": "K steps replayed from one CUDA graph"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"],
                         "unit": "GB/s", "frac": achieved / pk["hbm_gbs"],
                         "peak_kind": pk["hbm_kind"],
                         "traffic": ncu.get("cfg2_traffic_bytes"),
                         "bytes_alg_per_launch": B_ALG * shard,
                         "kernel_ms": r["kernel_ms"],
                         "fp64_pipe_frac": ncu.get("cfg2_fp64_pipe_frac"),
                         "fp64_peak_tflops": pk["fp64_tflops"],
                         "fp64_note": "measured DFMA peak (profiles/r02_ubench_fp64.json); "
                                      "fp64_pipe_frac from the committed ncu capture"},
            "gpu_launches": engine.launches_per_step * args.steps,
            "clocks": r["clocks"],
            "gather": {"ms": r["gather_ms"], "to_rank": 0,
                       "bytes": int(BATCH * N_MODE * 16 * (world - 1) / world),
                       "how": f"torch.distributed gather ({engine.backend if world > 1 else 'none, one rank'}), "
                              "timed apart from the products"},
        }
        if "e2e_ms" in r:
            line["e2e"] = {"value": BATCH * args.steps / (r["e2e_ms"] * 1e-3), "unit": UNIT,
                           "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": r["d2h"],
                           "path": "batched.hankel_tvp_partial_host: pinned host -> host"}
        if "weak_ms_total" in r:
            line["weak"] = {"value": world * BATCH * args.steps / (r["weak_ms_total"] * 1e-3),
                            "unit": UNIT, "products_per_gpu": BATCH,
                            "ms_per_step": r["weak_ms_total"] / args.steps}
        if r["full"] is not None:
            line.update(parity_vs_golden(r["full"], BATCH))
        if world == 1 and not args.no_extras and hasattr(engine, "torch"):
            try:
                line["configs"] = other_configs(engine.torch, pk["hbm_gbs"])
            except Exception as exc:  # never lose the headline line
                line["configs"] = {"error": repr(exc)}
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_block(args, line.get("configs"))
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------- CPU baseline
def cpu_baseline_block(args, configs):
    from oracle import cpu_baseline as C

    cores = C.host_cores()
    if args.cpu_quick:
        rates = {"kind": C.impl_kind(), "cores": cores, "cpu_model": C.cpu_model(),
                 "numpy": np.__version__, "cfg2": C.cfg2_rates(cores, steps=1)}
    else:
        rates = C.all_config_rates(cores)
    c2 = rates["cfg2"]
    best = "pow2" if c2["pow2"]["all_cores"] >= c2["exact"]["all_cores"] else "exact"
    block = {
        "value": c2[best]["all_cores"], "unit": UNIT, "cores": cores, "kind": rates["kind"],
        "path": {"pow2": "reference cli._fast_product_padded (L=4096, cli.py:277-291)",
                 "exact": "reference HankelTensor.tvp_partial (L=d_H=4093, hankel.py:140-147)"}[best],
        "sample": f"the full 4096-product cfg2 batch split over {cores} processes "
                  "(best of 3 barrier-separated steps); 1-core rate from 48 products",
        "one_core": c2[best]["one_core"],
        "exact_all_cores": c2["exact"]["all_cores"], "exact_one_core": c2["exact"]["one_core"],
        "pow2_all_cores": c2["pow2"]["all_cores"], "pow2_one_core": c2["pow2"]["one_core"],
        "cpu_model": rates["cpu_model"], "numpy": rates["numpy"],
    }
    if "cfg1" in rates:
        block["per_config"] = {k: rates[k] for k in ("cfg1", "cfg3", "cfg4", "cfg5")}
        if isinstance(configs, dict):  # GPU vs CPU side by side for every config
            for k in ("cfg1", "cfg3", "cfg4", "cfg5"):
                if k in configs and isinstance(configs[k], dict):
                    configs[k]["cpu"] = rates[k]
    return block


def run_reference(args):
    """The reference CPU path on all host cores, rank 0 only."""
    from oracle import cpu_baseline as C

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cores = C.host_cores()
    units, ts = C.step_times("cfg2", "pow2", BATCH, cores, steps=args.warmup + args.steps)
    ts = ts[args.warmup:]
    value = units / statistics.median(ts)
    u_ex, ts_ex = C.step_times("cfg2", "exact", BATCH, cores, steps=2)
    exact = u_ex / min(ts_ex)
    kind = C.impl_kind()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(ts) * 1e3, "higher_is_better": True,
        "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": WORKLOAD, "batch": BATCH, "n": N_MODE, "order": ORDER,
                   "fft_len": FFT_LEN},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "path": "reference cli._fast_product_padded (pow2 L=4096)",
                         "sample": f"each step = the full 4096-product batch over {cores} "
                                   "processes (inputs built before the first barrier)",
                         "exact_all_cores": exact, "cpu_model": C.cpu_model(),
                         "numpy": np.__version__},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- other configs
B_ALG_CFG = {
    "cfg1": (298 + 100 + 100) * 8,
    "cfg2": B_ALG,
    "cfg2_c64": B_ALG // 2,
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
    # cfg2 in single precision (complex64 variant, FP32 arithmetic, tol 1e-4)
    g = np.load(os.path.join(golden, "cfg2.npz"))
    h, x = workloads.cfg2()
    dh = torch.from_numpy(h.astype(np.complex64)).cuda()
    dx = torch.from_numpy(x.astype(np.complex64)).cuda()
    y64 = torch.empty((h.shape[0], N_MODE), dtype=torch.complex64, device=dh.device)
    f2 = lambda: batched.hankel_tvp_partial(dh, [dx, dx, dx], (N_MODE,) * ORDER, out=y64)
    ms = _graph_ms(torch, f2, 20)
    y = y64.cpu().numpy()
    err = max(_relerr(y[s], g["y"][k]) for k, s in enumerate(g["sel"]))
    rec("cfg2_c64", h.shape[0], ms, err,
        {"metric_note": "cfg2 with complex64 inputs/outputs and FP32 arithmetic "
                        "(B_alg halves: 49,128 B/product); parity vs the reference's "
                        "complex128 outputs, north_star tolerance 1e-4"})
    del dh, dx, y64
    # cfg3: one large real product (four-step, L = 3072 x 4096: TMA column passes,
    # ping-pong row stage)
    g = np.load(os.path.join(golden, "cfg3.npz"))
    h, x = workloads.cfg3()
    dh = torch.from_numpy(h).cuda()[None]
    dx = torch.from_numpy(x).cuda()[None]
    f3 = lambda: batched.hankel_tvp_partial(dh, [dx, dx], (1 << 22,) * 3)
    ms = _dev_ms(torch, f3, 5)
    y = f3()[0].cpu().numpy()
    rec("cfg3", 1, ms, _relerr(y[g["idx"]], g["y"]))
    del dh, dx
    # cfg4: 1024 BHHB products, 2D block kernels (192-point columns x 256-point rows)
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
    g50 = np.load(os.path.join(golden, "cfg5_sweep50.npz"))
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
    U50 = floop()[:2].cpu().numpy()
    perr = max(_relerr(U50[s] @ U50[s].conj().T, g50[f"U50_{s}"] @ g50[f"U50_{s}"].conj().T)
               for s in range(2))
    rec("cfg5", sig.shape[0] * 25, ms, _relerr(T[g["rows"]], g["T1_rows"]),
        {"metric_note": "times_matrices step of one HOOI iteration (256 signals x 25 "
                        "products, cached spectra); per-iteration SVD excluded",
         "loop_50_sweeps_ms": ms_loop,
         "loop_products_per_s": sig.shape[0] * 25 * 50 / (ms_loop * 1e-3),
         "loop_U50_projector_rel_err": perr,
         "loop_parity_note": "signals 0,1 after 50 sweeps vs the reference's own loop "
                             "(tests/golden/cfg5_sweep50.npz)"})
    return out


# ---------------------------------------------------------------- launcher
def relaunch(args):
    """``--gpus N`` outside torchrun: re-launch under torch.distributed.run,
    one process per GPU, rendezvous on 127.0.0.1."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--engine", default="",
                    help="module:Class of an alternative product engine (tests use a CPU "
                         "engine to drive the multi-rank harness over gloo)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-quick", action="store_true",
                    help="cfg2-only CPU baseline (skip the per-config CPU columns)")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the cfg1/3/4/5 side measurements")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--ref-products-per-core", type=int, default=0,
                    help="(kept for compatibility; the CPU legs time the full batch)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
