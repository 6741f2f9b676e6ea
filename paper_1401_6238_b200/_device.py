"""Per-object device state for the numpy-facing drop-in classes.

Each structured tensor keeps, per CUDA device, its generating data and its
cached spectrum (the reference's ``cached_property`` spectrum,
hankel.py:37-40 / 126-128) resident in HBM.  Products upload the vectors,
launch the fused kernel on the current stream and copy the result back.
"""

from __future__ import annotations

import ctypes
import itertools
import threading

import numpy as np
import torch

from . import _native as N
from . import batched


_CUDA_OK = False


def require_cuda() -> int:
    global _CUDA_OK
    if not _CUDA_OK:
        if not torch.cuda.is_available():
            raise RuntimeError(
                "no CUDA device: the hankelfft_b200 product path runs only on the GPU "
                "(there is no CPU fallback)")
        _CUDA_OK = True
    return torch.cuda.current_device()


def _dedupe(arrays):
    """Map equal input arrays to one index (one device upload, one FFT).

    Identical vectors give bit-identical transforms, so merging them does not
    change the result.
    """
    uniq, idx = [], []
    for a in arrays:
        for k, u in enumerate(uniq):
            if a is u or (a.shape == u.shape and np.array_equal(a, u)):
                idx.append(k)
                break
        else:
            uniq.append(a)
            idx.append(len(uniq) - 1)
    return uniq, idx


def _upload(arrays, dev, add_batch=True):
    out = []
    for a in arrays:
        t = torch.from_numpy(np.ascontiguousarray(a)).to(f"cuda:{dev}")
        out.append(t.unsqueeze(0) if add_batch else t)
    return out


class _Staging:
    """Per-device pinned host + device scratch for numpy-facing calls.

    One pinned buffer receives all input vectors (one H2D copy), the result
    comes back through a pinned buffer (one D2H copy); the only host sync is
    the final stream synchronize.  Grows on demand, never shrinks.
    """

    _by_dev: dict = {}
    _by_dev_lock = threading.Lock()

    def __init__(self, dev):
        self.dev = dev
        self.cap = 0
        self.host = None
        self.devbuf = None
        # held from packing the inputs until the call's stream sync: the
        # buffers are shared by every numpy-facing call on this device
        self.lock = threading.RLock()

    @classmethod
    def get(cls, dev):
        st = cls._by_dev.get(dev)
        if st is None:
            with cls._by_dev_lock:
                st = cls._by_dev.get(dev)
                if st is None:
                    st = cls._by_dev[dev] = cls(dev)
        return st

    def ensure(self, n):
        if n > self.cap:
            cap = max(n, 2 * self.cap, 4096)
            self.host = torch.empty(cap, dtype=torch.complex128, pin_memory=True)
            self.devbuf = torch.empty(cap, dtype=torch.complex128, device=f"cuda:{self.dev}")
            self.cap = cap
            # cached views / addresses for the latency path
            self.hnp = self.host.numpy()
            self.hbase = self.host.data_ptr()
            self.dbase = self.devbuf.data_ptr()
        return self.host, self.devbuf


def _upload_packed(arrays, dev):
    """Upload several 1-D complex arrays with one pinned H2D copy; returns
    (1, n) device views in the same order."""
    total = sum(a.shape[0] for a in arrays)
    host, devbuf = _Staging.get(dev).ensure(total)
    hnp = host.numpy()
    off = 0
    for a in arrays:
        hnp[off:off + a.shape[0]] = a
        off += a.shape[0]
    devbuf[:total].copy_(host[:total], non_blocking=True)
    views, off = [], 0
    for a in arrays:
        views.append(devbuf[off:off + a.shape[0]].view(1, -1))
        off += a.shape[0]
    return views


def _download(t: torch.Tensor) -> np.ndarray:
    out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    out.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return out.numpy().copy()


class HankelDeviceCache:
    def __init__(self, shape, h):
        self.shape = tuple(shape)
        self.h = h
        self._per_dev = {}
        self._lean = {}  # dev -> (plan, operand struct of the latency path or None)

    def _state(self) -> tuple:
        dev = require_cuda()
        st = self._per_dev.get(dev)
        if st is None:
            dh = torch.from_numpy(np.ascontiguousarray(self.h)).to(f"cuda:{dev}").unsqueeze(0)
            spec = batched.hankel_spectrum(dh, self.shape)
            st = (dh, spec)
            self._per_dev[dev] = st
        return dev, st

    def _spec(self) -> tuple:
        dev, st = self._state()
        return dev, st[1]

    # Up to this FFT length a single product runs on the latency kernel
    # (hk_small.cu), which recomputes ifft(h~) next to the vector transforms
    # in the same Stockham stages; it reads h itself, not the cached spectrum.
    SMALL_L = 4096

    def tvp_partial(self, xs) -> np.ndarray:
        dev, (dh, spec) = self._state()
        uniq, idx = _dedupe(xs)
        lean = self._lean.get(dev)
        if lean is None:
            plan = batched.hankel_plan(self.shape, dev)
            if plan.workspace_per_item == 0:
                small = plan.fft_lens[0] <= self.SMALL_L
                src = dh if small else spec
                # the operand struct and plan handle of the latency path, built once
                hop = N.Operand(src.data_ptr(), src.stride(0),
                                N.HK_C128 if small else N.HK_SPEC, 0)
                lean = self._lean[dev] = (plan, hop)
            else:
                lean = self._lean[dev] = (plan, None)
        plan, hop = lean
        if hop is not None:
            st = _Staging.get(dev)
            with st.lock:
                return self._lean_locked(st, dev, plan, hop, uniq, idx)
        with _Staging.get(dev).lock:
            up = _upload_packed(uniq, dev)
            y = batched.hankel_tvp_partial(spec, [up[i] for i in idx], self.shape, spectrum=True)
            return _download(y[0])

    def _lean_locked(self, st, dev, plan, hop, uniq, idx) -> np.ndarray:
        """Latency path: the vectors packed into one pinned buffer, one C-ABI
        call (zero-copy product or H2D + product + D2H) and one stream sync,
        with the plan and operand structs cached per device."""
        n_in = sum(a.shape[0] for a in uniq)
        n1 = self.shape[0]
        st.ensure(n_in + n1)
        hnp = st.hnp
        offs, off = [], 0
        for a in uniq:
            hnp[off:off + a.shape[0]] = a
            offs.append(off)
            off += a.shape[0]
        stream = torch.cuda.current_stream(dev)
        xoff = (ctypes.c_int64 * len(idx))(*[offs[i] for i in idx])
        dbase, hbase = st.dbase, st.hbase
        N.check(N.load_library().hk_tvp_partial_host(
            plan.handle, hop, hbase, n_in, xoff, len(idx), dbase, dbase + 16 * n_in,
            hbase + 16 * n_in, ctypes.c_void_p(stream.cuda_stream)), "hk_tvp_partial_host")
        return hnp[n_in:n_in + n1].copy()

    def tvp_full(self, xs) -> complex:
        dev, (dh, spec) = self._state()
        uniq, idx = _dedupe(xs)
        plan = batched.hankel_plan(self.shape, dev)
        with _Staging.get(dev).lock:
            up = _upload_packed(uniq, dev)
            if plan.workspace_per_item == 0 and plan.fft_lens[0] <= self.SMALL_L:
                a = batched.hankel_tvp_full(dh, [up[i] for i in idx], self.shape)
            else:
                a = batched.hankel_tvp_full(spec, [up[i] for i in idx], self.shape,
                                            spectrum=True)
            return complex(_download(a)[0])

    def times_matrices(self, mats) -> np.ndarray:
        dev, spec = self._spec()
        uniq, idx = _dedupe(mats)
        up = _upload(uniq, dev)
        T = batched.times_matrices(spec, self.shape, [up[i] for i in idx], spectrum=True)
        return T[0].cpu().numpy()


class BhhbDeviceCache:
    """Device state of a BHHB tensor routed to the native 2D block kernels."""

    def __init__(self, order, block_shape, outer_shape, H):
        self.order = order
        self.block_shape = tuple(block_shape)
        self.outer_shape = tuple(outer_shape)
        self.H = H
        self._per_dev = {}

    def _H(self):
        dev = require_cuda()
        dH = self._per_dev.get(dev)
        if dH is None:
            dH = torch.from_numpy(np.ascontiguousarray(self.H)).to(f"cuda:{dev}").unsqueeze(0)
            self._per_dev[dev] = dH
        return dev, dH

    def native_supported(self) -> bool:
        """True when the native 2D block plan covers this generator."""
        dev = require_cuda()
        try:
            batched.bhhb_plan(self.order, self.block_shape, self.outer_shape, dev)
        except NotImplementedError:
            return False
        return True

    def times_matrices(self, mats) -> np.ndarray:
        dev, dH = self._H()
        uniq, idx = _dedupe(mats)
        up = _upload(uniq, dev)
        T = batched.bhhb_times_matrices(dH, [up[i] for i in idx], self.order, self.block_shape,
                                        self.outer_shape)
        return T[0].cpu().numpy()

    def tvp_partial(self, xs) -> np.ndarray:
        dev, dH = self._H()
        uniq, idx = _dedupe(xs)
        up = _upload(uniq, dev)
        y = batched.bhhb_tvp_partial(dH, [up[i] for i in idx], self.order, self.block_shape,
                                     self.outer_shape)
        return y[0].cpu().numpy()

    def tvp_full(self, xs) -> complex:
        dev, dH = self._H()
        uniq, idx = _dedupe(xs)
        up = _upload(uniq, dev)
        a = batched.bhhb_tvp_full(dH, [up[i] for i in idx], self.order, self.block_shape,
                                  self.outer_shape)
        return complex(a[0].item())


def generic_times_matrices(tensor, mats) -> np.ndarray:
    """Column-combination loop of hankel.py:189-194 over any tensor exposing
    ``mode_sizes`` and ``tvp_partial`` (block tensors)."""
    sizes = tensor.mode_sizes
    ranks = tuple(M.shape[1] for M in mats)
    out = np.empty((sizes[0],) + ranks, dtype=np.complex128)
    for combo in itertools.product(*(range(r) for r in ranks)):
        cols = [M[:, j] for M, j in zip(mats, combo)]
        out[(slice(None),) + combo] = tensor.tvp_partial(cols)
    return out
