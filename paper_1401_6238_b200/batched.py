"""Batched device API over torch CUDA tensors (the engine under the drop-in).

Every function here launches the sm_100a kernels of ``libhankelfft_b200.so``
asynchronously on the current torch CUDA stream and returns device tensors;
nothing synchronises.  Inputs are complex128 (or float64, promoted on the fly
like the reference's ``core.as_complex``, core.py:21-22).  The products also
take complex64 / float32 operands (all of them single precision): FP32
arithmetic, complex64 results, relative error <= 1e-4 (the north_star's fp32
tolerance); on-chip lengths (d_H <= 8192), ``hankel_tvp_partial`` and
``hankel_tvp_full``.

Shapes (B = batch of independent tensors):
  h     : (B, d_H) generating vectors, or (B, L) spectra from ``hankel_spectrum``
  xs[p] : (B, n_{p+2}) for partial products, (B, n_{p+1}) for full products;
          passing the SAME tensor object twice means "same vector" (one FFT).
"""

from __future__ import annotations

import ctypes
import threading

import torch

from . import _native as N


def _require_cuda(t: torch.Tensor, name: str) -> None:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU path exists)")


def _physical(t: torch.Tensor) -> torch.Tensor:
    """Materialise torch's lazy conjugate / negative bits: the kernels read raw
    memory, and ``x.conj().contiguous()`` of a contiguous x is still a lazy view."""
    if t.is_conj():
        t = t.resolve_conj()
    if t.is_neg():
        t = t.resolve_neg()
    return t


def _operand(t: torch.Tensor, name: str, spectrum: bool = False) -> N.Operand:
    _require_cuda(t, name)
    if t.is_conj() or t.is_neg():
        raise ValueError(f"{name}: lazy conj/neg view reached the C ABI (call _physical)")
    if t.dim() != 2:
        raise ValueError(f"{name} must be 2-D (batch, length)")
    if t.stride(1) != 1:
        raise ValueError(f"{name} must be contiguous along its last dimension")
    if t.dtype == torch.complex128:
        dt = N.HK_SPEC if spectrum else N.HK_C128
    elif t.dtype == torch.float64 and not spectrum:
        dt = N.HK_F64
    elif t.dtype == torch.complex64 and not spectrum:
        dt = N.HK_C64
    elif t.dtype == torch.float32 and not spectrum:
        dt = N.HK_F32
    else:
        raise ValueError(f"{name} must be complex128{'' if spectrum else ', float64, complex64 or float32'}")
    return N.Operand(t.data_ptr(), t.stride(0), dt, 0)


def _out_dtype(h: torch.Tensor):
    """complex64 results for the single-precision variant (h complex64 / float32,
    FP32 arithmetic, north_star tolerance 1e-4), complex128 otherwise."""
    return torch.complex64 if h.dtype in (torch.complex64, torch.float32) else torch.complex128


def _stream(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _dev_index(t: torch.Tensor) -> int:
    return t.device.index if t.device.index is not None else torch.cuda.current_device()


def hankel_plan(shape, device: int, fft_len: int = 0) -> N.Plan:
    return N.hankel_plan(shape, device, fft_len)


class _NoWorkspace:
    """On-chip plans need no workspace: the C ABI receives NULL."""

    @staticmethod
    def data_ptr() -> int:
        return 0


def _workspace(plan: N.Plan, batch: int, device):
    """Caller-owned device workspace (two-level plans; NULL for on-chip plans).

    Freed by the caching allocator after the call: the stream-ordered reuse
    rule keeps it valid for the kernels already queued on this stream."""
    if plan.workspace_per_item == 0:
        return _NoWorkspace
    nbytes = int(N.load_library().hk_workspace_bytes(plan.handle, batch))
    return torch.empty((max(nbytes, 16),), dtype=torch.uint8, device=device)


class _OnDevice:
    """``torch.cuda.device(dev)`` only when ``dev`` is not already current
    (entering the context costs microseconds on the latency path)."""

    __slots__ = ("dev", "ctx")

    def __init__(self, dev: int):
        self.dev = dev
        self.ctx = None

    def __enter__(self):
        if torch.cuda.current_device() != self.dev:
            self.ctx = torch.cuda.device(self.dev)
            self.ctx.__enter__()
        return self

    def __exit__(self, *exc):
        if self.ctx is not None:
            self.ctx.__exit__(*exc)
        return False


def hankel_spectrum(h: torch.Tensor, shape, fft_len: int = 0) -> torch.Tensor:
    """Batched cached spectrum S = ifft(h~) (reference hankel.py:37-40, 126-128).

    Returns (B, L) complex128 in the library's internal layout (opaque: only
    meaningful as the ``h`` argument of the product functions).
    """
    h = _physical(h)
    dev = _dev_index(h)
    with _OnDevice(dev):
        plan = hankel_plan(shape, dev, fft_len)
        B = h.shape[0]
        spec = torch.empty((B, plan.spectrum_len), dtype=torch.complex128, device=h.device)
        ws = _workspace(plan, B, h.device)
        N.check(N.load_library().hk_spectrum(plan.handle, _operand(h, "h"), B, spec.data_ptr(),
                                             ws.data_ptr(), _stream(dev)), "hk_spectrum")
    return spec


def _physical_list(ts):
    """_physical over a list, preserving object identity of repeated entries
    (the same tensor twice still means "same vector")."""
    out, seen = [], {}
    for t in ts:
        key = id(t)
        if key not in seen:
            seen[key] = _physical(t)
        out.append(seen[key])
    return out


def _vector_operands(xs, names):
    ops = (N.Operand * len(xs))()
    for i, x in enumerate(xs):
        ops[i] = _operand(x, names[i])
    return ops


def hankel_tvp_partial(h: torch.Tensor, xs, shape, *, spectrum: bool = False,
                       out: torch.Tensor | None = None, fft_len: int = 0) -> torch.Tensor:
    """y_b = H_b x_{b,2} ... x_{b,m} (reference hankel.py:140-147), batched.

    Returns (B, n_1) complex128.  ``spectrum=True`` means ``h`` holds cached
    spectra from :func:`hankel_spectrum` with the same shape/fft_len.
    """
    shape = tuple(int(n) for n in shape)
    m = len(shape)
    xs = _physical_list(xs)
    h = _physical(h)
    if len(xs) != m - 1:
        raise ValueError(f"expected {m - 1} vectors, got {len(xs)}")
    dev = _dev_index(h)
    B = h.shape[0]
    with _OnDevice(dev):
        plan = hankel_plan(shape, dev, fft_len)
        if out is None:
            out = torch.empty((B, shape[0]), dtype=_out_dtype(h), device=h.device)
        _require_cuda(out, "out")
        if out.dtype != _out_dtype(h) or out.stride(-1) != 1:
            raise ValueError(f"out must be a {_out_dtype(h)} tensor contiguous along its rows")
        ops = _vector_operands(xs, [f"xs[{i}]" for i in range(len(xs))])
        ws = _workspace(plan, B, h.device)
        N.check(N.load_library().hk_tvp_partial(
            plan.handle, _operand(h, "h", spectrum), ops, len(xs), B, out.data_ptr(),
            out.stride(0), ws.data_ptr(), _stream(dev)), "hk_tvp_partial")
    return out


def hankel_tvp_full(h: torch.Tensor, xs, shape, *, spectrum: bool = False,
                    fft_len: int = 0) -> torch.Tensor:
    """alpha_b = H_b x_1 ... x_m, unconjugated (reference hankel.py:149-154). (B,) complex128."""
    shape = tuple(int(n) for n in shape)
    m = len(shape)
    xs = _physical_list(xs)
    h = _physical(h)
    if len(xs) != m:
        raise ValueError(f"expected {m} vectors, got {len(xs)}")
    dev = _dev_index(h)
    B = h.shape[0]
    with _OnDevice(dev):
        plan = hankel_plan(shape, dev, fft_len)
        alpha = torch.empty((B,), dtype=_out_dtype(h), device=h.device)
        ops = _vector_operands(xs, [f"xs[{i}]" for i in range(len(xs))])
        ws = _workspace(plan, B, h.device)
        N.check(N.load_library().hk_tvp_full(
            plan.handle, _operand(h, "h", spectrum), ops, len(xs), B, alpha.data_ptr(),
            ws.data_ptr(), _stream(dev)), "hk_tvp_full")
    return alpha


def _times_matrices_plan(plan, h, mats, sizes, n1, spectrum, what):
    """hk_times_matrices on an existing plan; mats[p] (B, sizes[p], R_p)."""
    mats = _physical_list(mats)
    h = _physical(h)
    dev = _dev_index(h)
    B = h.shape[0]
    for p, M in enumerate(mats):
        _require_cuda(M, f"mats[{p}]")
        if M.dim() != 3 or M.shape[1] != sizes[p] or M.dtype != torch.complex128:
            raise ValueError(f"matrix {p} must be (B, {sizes[p]}, R) complex128")
        if M.stride(2) != 1 or M.stride(1) != M.shape[2]:
            raise ValueError(f"matrix {p} must be row-major contiguous per item")
    ranks = [int(M.shape[2]) for M in mats]
    lib = N.load_library()
    r_arr = N.i64_array(ranks)
    ws_bytes = lib.hk_times_matrices_workspace_bytes(plan.handle, r_arr, len(mats), B)
    ws = torch.empty((max(int(ws_bytes), 16),), dtype=torch.uint8, device=h.device)
    T = torch.empty((B, n1, *ranks), dtype=torch.complex128, device=h.device)
    ptrs = (ctypes.c_void_p * len(mats))(*[M.data_ptr() for M in mats])
    strides = N.i64_array([M.stride(0) for M in mats])
    N.check(lib.hk_times_matrices(plan.handle, _operand(h, "h", spectrum), ptrs, strides,
                                  r_arr, len(mats), B, T.data_ptr(),
                                  T[0].numel() if B else 0, ws.data_ptr(), _stream(dev)), what)
    return T


def bhhb_times_matrices(H: torch.Tensor, mats, order, block_shape, outer_shape) -> torch.Tensor:
    """Batched BHHB T_b[:, j_2..j_m] = H_b x_2 M_2[:, j_2] ... (hankel.py:174-194 over
    block.py:136-144).  H: (B, d_in, d_out); mats[p]: (B, n_{p+2} N_{p+2}, R_p)
    whose rows are column-stacked (F-order) block vectors.  Returns
    (B, n_1 N_1, R_2, ..., R_m) complex128 (two-level 2D plans only)."""
    block_shape, outer_shape = tuple(block_shape), tuple(outer_shape)
    if len(mats) != order - 1:
        raise ValueError(f"expected {order - 1} matrices, got {len(mats)}")
    dev = _dev_index(H)
    with _OnDevice(dev):
        plan = bhhb_plan(order, block_shape, outer_shape, dev)
        Hf = _physical(H).reshape(H.shape[0], -1)
        sizes = [block_shape[p] * outer_shape[p] for p in range(1, order)]
        return _times_matrices_plan(plan, Hf, mats, sizes, block_shape[0] * outer_shape[0],
                                    False, "hk_times_matrices(block)")


def times_matrices(h: torch.Tensor, shape, mats, *, spectrum: bool = False,
                   fft_len: int = 0) -> torch.Tensor:
    """T_b[:, j_2..j_m] = H_b x_2 M_2[:, j_2] ... (reference hankel.py:174-194).

    mats[p]: (B, n_{p+2}, R_p) complex128 (row-major per item).  Passing the
    same tensor object for several modes shares its column spectra.
    Returns (B, n_1, R_2, ..., R_m) complex128.
    """
    shape = tuple(int(n) for n in shape)
    m = len(shape)
    if len(mats) != m - 1:
        raise ValueError(f"expected {m - 1} matrices, got {len(mats)}")
    dev = _dev_index(h)
    with _OnDevice(dev):
        plan = hankel_plan(shape, dev, fft_len)
        return _times_matrices_plan(plan, h, mats, shape[1:], shape[0], spectrum,
                                    "hk_times_matrices")


def _block_operand(t: torch.Tensor, name: str, length: int, spectrum: bool = False):
    """(B, length) vectors or (B, rows, cols) generators flattened per item."""
    _require_cuda(t, name)
    flat = t.reshape(t.shape[0], -1)
    if flat.shape[1] != length:
        raise ValueError(f"{name} must have {length} entries per item")
    return _operand(flat, name, spectrum), flat


def bhhb_plan(order, block_shape, outer_shape, device: int, fft_lens=None) -> N.Plan:
    return N.block_plan(order, (tuple(block_shape), tuple(outer_shape)), device, fft_lens)


def bhhb_tvp_partial(H: torch.Tensor, xs, order, block_shape, outer_shape, *,
                     spectrum: bool = False, out: torch.Tensor | None = None,
                     fft_lens=None) -> torch.Tensor:
    """Batched BHHB product y_b = vec(fft2(ifft2(H_b) .* prod fft2(X~_bp))[:n_1, :N_1])
    (reference block.py:136-144).

    H: (B, d_in, d_out) generating matrices (rows = inner index sums);
    xs[p]: (B, n_{p+1} * N_{p+1}) column-stacked (F-order) vectors.
    Returns (B, n_1 * N_1) complex128 column-stacked outputs.
    """
    block_shape, outer_shape = tuple(block_shape), tuple(outer_shape)
    xs = _physical_list(xs)
    H = _physical(H)
    if len(xs) != order - 1:
        raise ValueError(f"expected {order - 1} vectors, got {len(xs)}")
    dev = _dev_index(H)
    B = H.shape[0]
    with _OnDevice(dev):
        plan = bhhb_plan(order, block_shape, outer_shape, dev, fft_lens)
        hop, _ = _block_operand(H, "H", plan.spectrum_len if spectrum else
                                (sum(block_shape) - order + 1) * (sum(outer_shape) - order + 1),
                                spectrum)
        ops = (N.Operand * len(xs))()
        keep = []
        for i, x in enumerate(xs):
            ops[i], f = _block_operand(x, f"xs[{i}]", block_shape[i + 1] * outer_shape[i + 1])
            keep.append(f)
        n1 = block_shape[0] * outer_shape[0]
        if out is None:
            out = torch.empty((B, n1), dtype=torch.complex128, device=H.device)
        ws = _workspace(plan, B, H.device)
        N.check(N.load_library().hk_tvp_partial(plan.handle, hop, ops, len(xs), B,
                                                out.data_ptr(), out.stride(0), ws.data_ptr(),
                                                _stream(dev)), "hk_tvp_partial(block)")
    return out


def bhhb_tvp_full(H: torch.Tensor, xs, order, block_shape, outer_shape) -> torch.Tensor:
    """alpha_b = sum(ifft2(H_b) .* prod fft2(X~_bp)), unconjugated (block.py:146-153)."""
    block_shape, outer_shape = tuple(block_shape), tuple(outer_shape)
    xs = _physical_list(xs)
    H = _physical(H)
    if len(xs) != order:
        raise ValueError(f"expected {order} vectors, got {len(xs)}")
    dev = _dev_index(H)
    B = H.shape[0]
    with _OnDevice(dev):
        plan = bhhb_plan(order, block_shape, outer_shape, dev)
        hop, _ = _block_operand(
            H, "H", (sum(block_shape) - order + 1) * (sum(outer_shape) - order + 1))
        ops = (N.Operand * len(xs))()
        keep = []
        for i, x in enumerate(xs):
            ops[i], f = _block_operand(x, f"xs[{i}]", block_shape[i] * outer_shape[i])
            keep.append(f)
        alpha = torch.empty((B,), dtype=torch.complex128, device=H.device)
        ws = _workspace(plan, B, H.device)
        N.check(N.load_library().hk_tvp_full(plan.handle, hop, ops, len(xs), B,
                                             alpha.data_ptr(), ws.data_ptr(), _stream(dev)),
                "hk_tvp_full(block)")
    return alpha


def hankel_tvp_partial_multi(h: torch.Tensor, xs, shape, *, devices=None, gather_to=None,
                             fft_len: int = 0):
    """Batched H x_2 ... x_m sharded over several GPUs from ONE process
    (SURVEY §8e): contiguous shards of the batch (``dist.shard_range``), each
    launched on its device's current stream with no cross-device traffic
    except moving the shard's inputs there and -- only when ``gather_to`` is
    given -- the results back (peer copies over NVLink).

    h: (B, d_H), xs[p]: (B, n_{p+2}) on the host (pinned for async copies) or on
    any CUDA device; the same tensor object twice means the same vector.
    ``devices``: list of CUDA device indices (default: all visible).
    Returns the list of per-device (B_k, n_1) outputs (a Shard(0) layout), or
    one (B, n_1) tensor on ``gather_to``.  Nothing synchronises.
    """
    from .dist import shard_range

    shape = tuple(int(n) for n in shape)
    xs = list(xs)
    if len(xs) != len(shape) - 1:
        raise ValueError(f"expected {len(shape) - 1} vectors, got {len(xs)}")
    devices = list(range(torch.cuda.device_count())) if devices is None else list(devices)
    if not devices:
        raise RuntimeError("no CUDA device: the product path runs only on the GPU")
    B = h.shape[0]
    outs = []
    for k, dev in enumerate(devices):
        lo, hi = shard_range(B, k, len(devices))
        with torch.cuda.device(dev):
            if hi == lo:
                outs.append(torch.empty((0, shape[0]), dtype=torch.complex128,
                                        device=f"cuda:{dev}"))
                continue
            hs = h[lo:hi].to(f"cuda:{dev}", non_blocking=True)
            moved = {}
            xsd = []
            for x in xs:
                if id(x) not in moved:
                    moved[id(x)] = x[lo:hi].to(f"cuda:{dev}", non_blocking=True)
                xsd.append(moved[id(x)])
            outs.append(hankel_tvp_partial(hs, xsd, shape, fft_len=fft_len))
    if gather_to is None:
        return outs
    dst = torch.device(gather_to) if not isinstance(gather_to, int) else \
        torch.device("cuda", gather_to)
    return torch.cat([o.to(dst, non_blocking=True) for o in outs], dim=0)


class _HostPipeline:
    """Per-(device, shape) double-buffered device staging for host-buffer calls.

    ``lock`` is held while one call enqueues its chunks: the staging buffers
    and streams are shared by every host thread using this key, and the
    stream order then keeps one call's copies and kernels from touching
    another's buffers."""

    def __init__(self, dev, d, ns, n1, chunk, real_h, real_x):
        self.lock = threading.Lock()
        self.streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
        hd = torch.float64 if real_h else torch.complex128
        xd = torch.float64 if real_x else torch.complex128
        self.bufs = []
        for _ in range(2):
            self.bufs.append(dict(
                h=torch.empty((chunk, d), dtype=hd, device=dev),
                xs=[torch.empty((chunk, n), dtype=xd, device=dev) for n in ns],
                y=torch.empty((chunk, n1), dtype=torch.complex128, device=dev)))


_pipelines: dict = {}
_pipelines_lock = threading.Lock()


def hankel_tvp_partial_host(h: torch.Tensor, xs, shape, *, out: torch.Tensor | None = None,
                            chunk: int = 512) -> torch.Tensor:
    """Batched H x_2 ... x_m from HOST memory to HOST memory.

    h: (B, d_H) and xs[p]: (B, n_{p+2}) CPU tensors (pinned for full PCIe
    speed; the same tensor object twice = same vector).  Chunks of ``chunk``
    products are streamed through two CUDA streams so host->device copies,
    the fused kernel and device->host copies of consecutive chunks overlap.
    Returns a (B, n_1) complex128 CPU tensor (pinned).  The work is ordered
    before any later work on the current stream; synchronise before reading.
    """
    shape = tuple(int(n) for n in shape)
    xs = list(xs)
    if len(xs) != len(shape) - 1:
        raise ValueError(f"expected {len(shape) - 1} vectors, got {len(xs)}")
    dev = torch.cuda.current_device()
    B = h.shape[0]
    uniq, idx = [], []
    for x in xs:
        for k, u in enumerate(uniq):
            if x is u:
                idx.append(k)
                break
        else:
            uniq.append(x)
            idx.append(len(uniq) - 1)
    ns = [int(u.shape[1]) for u in uniq]
    real_h = h.dtype == torch.float64
    real_x = all(u.dtype == torch.float64 for u in uniq)
    key = (dev, shape, int(h.shape[1]), tuple(ns), chunk, real_h, real_x)
    with _pipelines_lock:
        pipe = _pipelines.get(key)
        if pipe is None:
            pipe = _HostPipeline(dev, int(h.shape[1]), ns, shape[0], chunk, real_h, real_x)
            _pipelines[key] = pipe
    if out is None:
        out = torch.empty((B, shape[0]), dtype=torch.complex128, pin_memory=True)
    cur = torch.cuda.current_stream(dev)
    with pipe.lock:
        for s in pipe.streams:
            s.wait_stream(cur)
        for c, start in enumerate(range(0, B, chunk)):
            nb = min(chunk, B - start)
            st, buf = pipe.streams[c % 2], pipe.bufs[c % 2]
            with torch.cuda.stream(st):
                buf["h"][:nb].copy_(h[start:start + nb], non_blocking=True)
                for k, u in enumerate(uniq):
                    buf["xs"][k][:nb].copy_(u[start:start + nb], non_blocking=True)
                hankel_tvp_partial(buf["h"][:nb], [buf["xs"][i][:nb] for i in idx], shape,
                                   out=buf["y"][:nb])
                out[start:start + nb].copy_(buf["y"][:nb], non_blocking=True)
        for s in pipe.streams:
            cur.wait_stream(s)
    return out
