"""A CPU product engine for driving bench.py's multi-rank harness over gloo
in the CPU test suite (tests/test_bench_multirank.py).  It computes the cfg2
products with the oracle (test infrastructure), so the harness's sharding,
max-over-ranks timing, gather and golden parity check run end to end without
a GPU.  It is never used by the driver's runs."""

import time

import numpy as np
import torch

from oracle import hankel_oracle as O
from paper_1401_6238_b200 import workloads


class WallTimer:
    def start(self):
        self.t0 = time.perf_counter()

    def stop(self):
        self.t1 = time.perf_counter()

    def ms(self):
        return (self.t1 - self.t0) * 1e3


class CpuEngine:
    backend = "gloo"
    launches_per_step = 0
    dtype = "c128"

    def __init__(self, local_rank):
        self.torch = None  # no GPU side configs
        self.shape = (1024,) * 4

    def device(self):
        return torch.device("cpu")

    def load(self, lo, hi):
        import bench

        h, x = workloads.cfg2()  # the full seeded batch; the bench runs a prefix
        h, x = h[: bench.BATCH], x[: bench.BATCH]
        self.lo, self.hi = lo, hi
        self.h, self.x = h[lo:hi], x[lo:hi]
        self.y = torch.zeros((hi - lo, 1024), dtype=torch.complex128)

    def unload(self):
        pass

    def step(self):
        if self.hi > self.lo:
            y = O.hankel_tvp_partial_batch(self.h, [self.x] * 3, self.shape, length=4096)
            self.y = torch.from_numpy(np.ascontiguousarray(y))

    def sync(self):
        pass

    def timer(self):
        return WallTimer()

    def result(self):
        return self.y
