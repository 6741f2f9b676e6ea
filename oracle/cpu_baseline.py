"""CPU baselines of the reference path, timed on the host cores.

TEST / MEASUREMENT INFRASTRUCTURE ONLY: used by ``bench.py``'s cpu_baseline
leg and its ``--impl reference`` arm, never by the product package.

What is timed, per config, is the REFERENCE's own code path:

* ``kind = "reference"`` -- the unmodified reference package installed into
  ``baseline/_ref`` (``pip install --no-deps --target baseline/_ref``; it is
  git-ignored but travels to the GPU box), called through its public API
  exactly as a user would: ``HankelTensor(...).tvp_partial`` (exact
  embedding length d_H, hankel.py:140-147), ``cli._fast_product_padded``
  (its benchmark-only pow2 variant, cli.py:277-291), ``BhhbTensor`` and the
  HOOI loop ``times_matrices`` -> ``truncated_left_singular_vectors``
  (hankel.py:174-194, decompose.py:35-41);
* ``kind = "port"`` -- when baseline/_ref is absent, the pinned numpy
  restatement in ``oracle/hankel_oracle.py`` (same pocketfft calls).

Threads: OMP/OpenBLAS/MKL pinned to 1 thread, one spawned worker process per
core, each on a contiguous shard of the same seeded inputs; inputs are built
before a common start time and the clock covers the compute loop only.
Products/s are reported for 1 core and for all cores.
"""

from __future__ import annotations

import os
import platform
import statistics
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF_DIR = os.path.join(ROOT, "baseline", "_ref")

for _k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_k, "1")


def impl_kind() -> str:
    return "reference" if os.path.isfile(os.path.join(REF_DIR, "hankelfft", "__init__.py")) \
        else "port"


def _load():
    """(kind, ops) with ops a dict of callables over the chosen implementation."""
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    kind = impl_kind()
    if kind == "reference":
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        import hankelfft as R
        from hankelfft import cli as RC

        return kind, {
            "partial": lambda h, shape, xs: R.HankelTensor(shape, h).tvp_partial(xs),
            "partial_pow2": lambda h, shape, xs: RC._fast_product_padded(h, shape, xs),
            "bhhb": lambda H, block, outer, xs: R.BhhbTensor(len(block), block, outer,
                                                              H).tvp_partial(xs),
            "tensor": lambda shape, h: R.HankelTensor(shape, h),
            "times_matrices": lambda T, mats: R.times_matrices(T, mats),
            "tlsv": R.truncated_left_singular_vectors,
        }
    from oracle import hankel_oracle as O

    return kind, {
        "partial": O.hankel_tvp_partial,
        "partial_pow2": O.hankel_tvp_partial_padded,
        "bhhb": O.bhhb_tvp_partial,
        "tensor": lambda shape, h: (shape, h),
        "times_matrices": lambda T, mats: O.times_matrices(T[1], T[0], mats),
        "tlsv": O.truncated_left_singular_vectors,
    }


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ------------------------------------------------------------------ workers
def _inputs(cfg, lo, hi, variant):
    """Seeded inputs of products [lo, hi) of a config and the per-unit call."""
    from paper_1401_6238_b200 import workloads

    kind, ops = _load()
    if cfg == "cfg2":
        h, x = workloads.cfg2()
        h, x = h[lo:hi].copy(), x[lo:hi].copy()
        f = ops["partial_pow2" if variant == "pow2" else "partial"]
        shape = (1024,) * 4
        return hi - lo, lambda b: f(h[b], shape, [x[b]] * 3)
    if cfg == "cfg4":
        H, X = workloads.cfg4()
        H, X = H[lo:hi].copy(), X[lo:hi].copy()
        blk = (64,) * 3
        xv = [X[b].ravel(order="F") for b in range(hi - lo)]
        return hi - lo, lambda b: ops["bhhb"](H[b], blk, blk, [xv[b], xv[b]])
    if cfg == "cfg5":
        sig, U0, shape = workloads.cfg5(signals=hi)
        sig = sig[lo:hi]
        n = shape[0]

        def loop(s):
            T = ops["tensor"](shape, sig[s])
            U = U0
            for _ in range(50):
                Tm = ops["times_matrices"](T, [np.conj(U)] * 2)
                U = ops["tlsv"](Tm.reshape(n, -1), 5)
        return hi - lo, loop
    if cfg == "cfg1":
        h, x = workloads.cfg1()
        return hi - lo, lambda b: ops["partial"](h, (100,) * 3, [x, x])
    if cfg == "cfg3":
        h, x = workloads.cfg3()
        f = ops["partial_pow2" if variant == "pow2" else "partial"]
        return 1, lambda b: f(h, (1 << 22,) * 3, [x, x])
    raise ValueError(cfg)


def _worker(cfg, variant, lo, hi, steps, barrier, queue, per_call):
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    try:
        n, call = _inputs(cfg, lo, hi, variant)
        times = []
        for _ in range(steps):
            barrier.wait()
            if per_call:  # latency: median of single calls
                ts = []
                for b in range(n):
                    t0 = time.perf_counter()
                    call(b)
                    ts.append(time.perf_counter() - t0)
                times.append(statistics.median(ts))
            else:
                t0 = time.perf_counter()
                for b in range(n):
                    call(b)
                times.append(time.perf_counter() - t0)
        queue.put((lo, n, times))
    except BaseException as exc:  # never hang the barrier
        barrier.abort()
        queue.put((lo, -1, repr(exc)))


def _shards(total, cores):
    base, rem = divmod(total, cores)
    out, lo = [], 0
    for r in range(cores):
        hi = lo + base + (1 if r < rem else 0)
        if hi > lo:
            out.append((lo, hi))
        lo = hi
    return out


def step_times(cfg, variant, total, cores, steps=1, per_call=False, timeout=900):
    """Run `total` units of a config split over `cores` worker processes for
    `steps` barrier-separated steps.  Returns (units per step, [seconds per
    step]) with each step's time the max over workers (inputs are generated
    before the first barrier and not timed)."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    shards = _shards(total, cores)
    barrier = ctx.Barrier(len(shards))
    queue = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(cfg, variant, lo, hi, steps, barrier, queue,
                                               per_call), daemon=True)
             for lo, hi in shards]
    for p in procs:
        p.start()
    res = [queue.get(timeout=timeout) for _ in procs]
    for p in procs:
        p.join(timeout=30)
    bad = [r for r in res if r[1] < 0]
    if bad:
        raise RuntimeError(f"cpu baseline worker failed: {bad[0][2]}")
    units = sum(r[1] for r in res)
    per_step = [max(r[2][k] for r in res) for k in range(steps)]
    return units, per_step


def rate(cfg, variant, total, cores, steps=1):
    """Best-of-`steps` units/s of `total` units over `cores` workers."""
    units, ts = step_times(cfg, variant, total, cores, steps)
    t = min(ts)
    return units / t, units, t


def cfg2_rates(cores, variants=("pow2", "exact"), steps=3, one_core_sample=48):
    """cfg2 products/s per variant: the full 4096 batch on all cores, and a
    1-core sample."""
    out = {}
    for v in variants:
        r_all, units, wall = rate("cfg2", v, 4096, cores, steps)
        r_one, u1, w1 = rate("cfg2", v, one_core_sample, 1, 1)
        out[v] = {"all_cores": r_all, "one_core": r_one, "units": units, "wall_s": wall,
                  "one_core_units": u1}
    return out


def all_config_rates(cores):
    """Reference-path rates for cfg1..cfg5 (BASELINE.md §3 sample sizes; cfg3 one
    product per variant, cfg5 one signal per core)."""
    out = {"kind": impl_kind(), "cores": cores, "cpu_model": cpu_model(),
           "numpy": np.__version__, "python": platform.python_version()}
    out["cfg2"] = cfg2_rates(cores)
    # cfg1: median latency of 1000 calls, one core
    _, ts = step_times("cfg1", "exact", 1000, 1, 1, per_call=True)
    out["cfg1"] = {"exact": {"median_us_per_call": ts[0] * 1e6, "one_core": 1.0 / ts[0],
                             "calls": 1000}}
    r4, u4, w4 = rate("cfg4", "exact", 1024, cores)
    r4one, _, _ = rate("cfg4", "exact", 16, 1)
    out["cfg4"] = {"exact": {"all_cores": r4, "one_core": r4one, "units": u4, "wall_s": w4}}
    # cfg5: all 50 sweeps on one signal per core (signals are independent)
    units, ts = step_times("cfg5", "exact", cores, cores, 1)
    r5 = units * 50 * 25 / ts[0]
    out["cfg5"] = {"exact": {"all_cores": r5, "one_core": r5 / cores, "signals": units,
                             "wall_s": ts[0],
                             "note": "50 sweeps of times_matrices + SVD per signal; "
                                     "products/s = signals*50*25/wall"}}
    # cfg3: one product per variant (two single-core workers in turn)
    _, t3p = step_times("cfg3", "pow2", 1, 1, 1)
    _, t3e = step_times("cfg3", "exact", 1, 1, 1)
    out["cfg3"] = {"exact": {"seconds_per_product": t3e[0], "one_core": 1.0 / t3e[0]},
                   "pow2": {"seconds_per_product": t3p[0], "one_core": 1.0 / t3p[0]}}
    return out
