"""CPU oracle for the fast Hankel tensor-vector product path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline / ``--impl reference`` leg may use it, and only as the checker
(or as the timed reference CPU arm), never as the thing measured or shipped.

This is a numpy restatement of the reference ``hankelfft`` 0.1.0 algorithm
for the hot path (arXiv 1401.6238 Sec. 3).  Each function cites the
reference file:line it follows (paths relative to ``/root/reference/pkg``).
The FFT arithmetic itself lives in the reference's third-party dependency,
numpy's bundled pocketfft (``numpy>=1.24`` floor in ``pyproject.toml:11``;
numpy 2.3.5 in this image).  The oracle calls the same ``numpy.fft``
entry points with the same default ("backward") normalisation as
``src/hankelfft/fourier.py:28-49``: forward unnormalised, inverse 1/n.

Parity is PINNED: ``tests/test_oracle.py`` checks every function here
against (a) the known-answer vectors of the reference test-suite and (b)
golden outputs produced by running the reference itself in the build
container (``oracle/gen_golden.py`` -> ``tests/golden/*.npz``).
"""

from __future__ import annotations

import math
from functools import reduce

import numpy as np

#: core.py:17-18 -- refuse dense tensors above this many entries.
DENSE_CAP = 10_000_000


def c128(a) -> np.ndarray:
    """core.py:21-22 -- every input is promoted to complex128."""
    return np.asarray(a, dtype=np.complex128)


# --------------------------------------------------------------------------
# dense brute-force ground truth (core.py) -- O(n^m), small sizes only
# --------------------------------------------------------------------------

def _sum_grid(sizes):
    """Tensor of i_1 + ... + i_m over the index box (core.py:102-104)."""
    return reduce(np.add.outer, [np.arange(s) for s in sizes])


def _check_cap(shape, cap):
    if math.prod(shape) > cap:
        raise ValueError(f"dense tensor {tuple(shape)} exceeds cap {cap}")


def dense_hankel(h, shape, cap=DENSE_CAP):
    """A[i_1..i_m] = h[i_1+...+i_m]  (core.py:107-115)."""
    shape = tuple(int(s) for s in shape)
    _check_cap(shape, cap)
    return c128(h)[_sum_grid(shape)]


def dense_anticirculant(c, order, dim, cap=DENSE_CAP):
    """A[i] = c[(sum i) mod n]  (core.py:118-125)."""
    shape = (dim,) * order
    _check_cap(shape, cap)
    return c128(c)[_sum_grid(shape) % dim]


def _digit_sums(full_sizes, level_shapes):
    """Per level, the tensor of summed level digits (inner level fastest).

    Restates core.py:128-135 (two levels) and core.py:187-194 (k levels).
    """
    sums = []
    stride = [1] * len(full_sizes)
    for lv in level_shapes:
        digits = [(np.arange(full_sizes[p]) // stride[p]) % lv[p]
                  for p in range(len(full_sizes))]
        sums.append(reduce(np.add.outer, digits))
        stride = [stride[p] * lv[p] for p in range(len(full_sizes))]
    return sums


def dense_level_k(G, level_shapes, cap=DENSE_CAP):
    """Level-k block Hankel tensor from its generating tensor (core.py:170-195).

    Level 2 with (block, outer) is the BHHB tensor of core.py:138-155.
    """
    level_shapes = [tuple(int(s) for s in lv) for lv in level_shapes]
    m = len(level_shapes[0])
    full = tuple(math.prod(lv[p] for lv in level_shapes) for p in range(m))
    _check_cap(full, cap)
    return c128(G)[tuple(_digit_sums(full, level_shapes))]


def dense_bhhb(H, block, outer, cap=DENSE_CAP):
    """core.py:138-155."""
    return dense_level_k(H, [block, outer], cap)


def dense_baab(C, order, cap=DENSE_CAP):
    """Block anti-circulant with anti-circulant blocks (core.py:158-167)."""
    C = c128(C)
    n, N = C.shape
    full = (n * N,) * order
    _check_cap(full, cap)
    si, sj = _digit_sums(full, [(n,) * order, (N,) * order])
    return C[si % n, sj % N]


def brute_tvp_partial(A, xs):
    """Contract modes 2..m with vectors, last mode first (core.py:54-69)."""
    out = c128(A)
    for x in reversed([c128(x) for x in xs]):
        out = out @ x
    return out


def brute_tvp_full(A, xs):
    """core.py:72-79 -- x_1^T (A x_2 ... x_m), unconjugated."""
    xs = [c128(x) for x in xs]
    return complex(np.dot(xs[0], brute_tvp_partial(A, xs[1:])))


def brute_mode_product(A, axis, M):
    """(A x_axis M)[..j..] = sum_i A[..i..] M[i, j]  (core.py:34-51)."""
    out = np.tensordot(c128(A), c128(M), axes=([axis], [0]))
    return np.moveaxis(out, -1, axis)


# --------------------------------------------------------------------------
# FFT fast path, exactly as the reference evaluates it
# --------------------------------------------------------------------------

def acirc_spectrum(c):
    """diag(D) = ifft(c)  (hankel.py:37-40 -> fourier.py:32-33)."""
    return np.fft.ifft(c128(c))


def _spectral_product(spec, xhats):
    """buf = spectrum.copy(); buf *= fft(x) per vector, in order (hankel.py:61-71)."""
    buf = spec.copy()
    for xh in xhats:
        buf *= xh
    return buf


def acirc_tvp_partial(c, xs):
    """y = fft(ifft(c) .* fft(x_2) ... .* fft(x_m))  (hankel.py:42-45)."""
    spec = acirc_spectrum(c)
    return np.fft.fft(_spectral_product(spec, [np.fft.fft(c128(x)) for x in xs]))


def acirc_tvp_full(c, xs):
    """alpha = ifft(c)^T (fft(x_1) .* ... .* fft(x_m)), no conjugation (hankel.py:47-59)."""
    spec = acirc_spectrum(c)
    buf = np.ones(spec.shape[0], dtype=np.complex128)
    for x in xs:
        buf *= np.fft.fft(c128(x))
    return complex(np.dot(spec, buf))


def _zero_pad(x, length):
    """hankel.py:130-138 -- zero-pad a mode vector to the embedding length."""
    x = c128(x)
    out = np.zeros(x.shape[:-1] + (length,), dtype=np.complex128)
    out[..., : x.shape[-1]] = x
    return out


def hankel_dof(shape):
    """d_H = n_1 + ... + n_m - m + 1  (hankel.py:108-111)."""
    return sum(shape) - len(shape) + 1


def hankel_tvp_partial(h, shape, xs):
    """H x_2 ... x_m via the exact-length anti-circulant embedding (hankel.py:140-147)."""
    d = hankel_dof(shape)
    padded = [_zero_pad(x, d) for x in xs]
    return acirc_tvp_partial(h, padded)[: shape[0]]


def hankel_tvp_full(h, shape, xs):
    """H x_1 ... x_m  (hankel.py:149-154)."""
    d = hankel_dof(shape)
    return acirc_tvp_full(h, [_zero_pad(x, d) for x in xs])


def hankel_tvp_partial_padded(h, shape, xs, length=None):
    """Power-of-two embedding length variant (cli.py:277-291).

    Any length >= d_H gives the same tensor product (no index sum reaches
    the wrap-around), which is what the GPU path exploits.
    """
    d = hankel_dof(shape)
    if length is None:
        length = 1 << max(0, (d - 1).bit_length())
    return acirc_tvp_partial(_zero_pad(h, length),
                             [_zero_pad(x, length) for x in xs])[: shape[0]]


def hankel_tvp_partial_batch(h, xs, shape, length=None):
    """Batched restatement of hankel.py:140-147 (rows are independent products).

    h: (B, d_H); xs: list of m-1 arrays (B, n_p).  With length=None the exact
    embedding length d_H is used, like the reference; the FFT of every
    vector is taken separately (the reference does not deduplicate).
    """
    d = hankel_dof(shape)
    L = d if length is None else length
    spec = np.fft.ifft(_zero_pad(h, L), axis=-1)
    buf = spec
    for x in xs:
        buf = buf * np.fft.fft(_zero_pad(x, L), axis=-1)
    return np.fft.fft(buf, axis=-1)[..., : shape[0]]


def times_matrices(h, shape, mats):
    """Column-by-column tensor-matrix product over modes 2..m (hankel.py:174-194)."""
    mats = [c128(M) for M in mats]
    ranks = tuple(M.shape[1] for M in mats)
    out = np.empty((shape[0],) + ranks, dtype=np.complex128)
    for combo in np.ndindex(*ranks):
        cols = [M[:, j] for M, j in zip(mats, combo)]
        out[(slice(None),) + combo] = hankel_tvp_partial(h, shape, cols)
    return out


def times_matrices_fast(h, shape, mats, length=None):
    """Same product as :func:`times_matrices`, vectorised over column combos.

    Used to time/check cfg5 at size; column spectra are taken once.
    """
    d = hankel_dof(shape)
    L = d if length is None else length
    mats = [c128(M) for M in mats]
    spec = np.fft.ifft(_zero_pad(h, L))
    colspec = [np.fft.fft(_zero_pad(M.T, L), axis=-1) for M in mats]   # (R_p, L)
    buf = spec
    for p, cs in enumerate(colspec):
        idx = [None] * len(mats)
        idx[p] = slice(None)
        buf = buf * cs[tuple(idx) + (slice(None),)]
    y = np.fft.fft(buf, axis=-1)[..., : shape[0]]          # (R_2, ..., R_m, n_1)
    return np.moveaxis(y, -1, 0)


# ---- block / multi-level (block.py) ---------------------------------------

def vec(M):
    """Column stacking (block.py:25-27)."""
    return np.asarray(M).ravel(order="F")


def unvec(v, rows, cols):
    """block.py:30-34."""
    v = c128(v)
    if v.shape != (rows * cols,):
        raise ValueError(f"vector must have length {rows * cols}, got {v.shape}")
    return v.reshape((rows, cols), order="F")


def bhhb_tvp_partial(H, block, outer, xs, as_matrix=False):
    """Ytilde = fft2(ifft2(H) .* prod fft2(Xtilde_p)); y = vec(corner) (block.py:136-144)."""
    H = c128(H)
    buf = np.fft.ifft2(H)
    for p, x in enumerate(xs):
        Xp = np.zeros(H.shape, dtype=np.complex128)
        n, N = block[p + 1], outer[p + 1]
        Xp[:n, :N] = unvec(x, n, N)                       # block.py:129-134
        buf = buf * np.fft.fft2(Xp)
    Y = np.fft.fft2(buf)[: block[0], : outer[0]]
    return Y if as_matrix else vec(Y)


def bhhb_tvp_partial_batch(H, X, block, outer):
    """Batched BHHB H x^2 for order 3 with the same x twice (cfg4).

    H: (B, d_in, d_out); X: (B, n, N) matrices (x = vec(X)); returns (B, n*N)
    F-order vectors.  Follows block.py:136-144 (two separate fft2's of x).
    """
    B, din, dout = H.shape
    buf = np.fft.ifft2(c128(H))
    Xp = np.zeros((B, din, dout), dtype=np.complex128)
    Xp[:, : X.shape[1], : X.shape[2]] = X
    for _ in range(len(block) - 1):
        buf = buf * np.fft.fft2(Xp)
    Y = np.fft.fft2(buf)[:, : block[0], : outer[0]]
    return np.transpose(Y, (0, 2, 1)).reshape(B, -1)


def bhhb_tvp_full(H, block, outer, xs):
    """alpha = sum_{jk} ifft2(H) .* prod fft2(Xtilde_p)  (block.py:146-153)."""
    H = c128(H)
    buf = np.fft.ifft2(H)
    for p, x in enumerate(xs):
        Xp = np.zeros(H.shape, dtype=np.complex128)
        n, N = block[p], outer[p]
        Xp[:n, :N] = unvec(x, n, N)
        buf = buf * np.fft.fft2(Xp)
    return complex(np.sum(buf))


def baab_tvp_partial(C, xs):
    """block.py:65-81 -- exact n x N circular products."""
    C = c128(C)
    n, N = C.shape
    buf = np.fft.ifft2(C)
    for x in xs:
        buf = buf * np.fft.fft2(unvec(x, n, N))
    return vec(np.fft.fft2(buf))


def baab_tvp_full(C, xs):
    """block.py:83-86."""
    C = c128(C)
    n, N = C.shape
    buf = np.fft.ifft2(C)
    for x in xs:
        buf = buf * np.fft.fft2(unvec(x, n, N))
    return complex(np.sum(buf))


def levelk_tvp_partial(G, level_shapes, xs):
    """block.py:214-238 -- fftn version, corner, F-order ravel."""
    G = c128(G)
    buf = np.fft.ifftn(G)
    for p, x in enumerate(xs):
        shp = tuple(lv[p + 1] for lv in level_shapes)
        X = np.zeros(G.shape, dtype=np.complex128)
        X[tuple(slice(0, s) for s in shp)] = c128(x).reshape(shp, order="F")
        buf = buf * np.fft.fftn(X)
    corner = tuple(slice(0, lv[0]) for lv in level_shapes)
    return np.fft.fftn(buf)[corner].ravel(order="F")


def levelk_tvp_full(G, level_shapes, xs):
    """block.py:240-247."""
    G = c128(G)
    buf = np.fft.ifftn(G)
    for p, x in enumerate(xs):
        shp = tuple(lv[p] for lv in level_shapes)
        X = np.zeros(G.shape, dtype=np.complex128)
        X[tuple(slice(0, s) for s in shp)] = c128(x).reshape(shp, order="F")
        buf = buf * np.fft.fftn(X)
    return complex(np.sum(buf))


# ---- HOOI pieces used by the cfg5 driver loop (decompose.py) ---------------

def fix_phase(U):
    """Largest-magnitude entry of each column made real positive (decompose.py:23-32)."""
    U = np.array(U, dtype=np.complex128, copy=True)
    for j in range(U.shape[1]):
        col = U[:, j]
        a = col[int(np.argmax(np.abs(col)))]
        if abs(a) > 0:
            U[:, j] = col * (np.conj(a) / abs(a))
    return U


def truncated_left_singular_vectors(M, r):
    """decompose.py:35-41."""
    U, _, _ = np.linalg.svd(c128(M), full_matrices=False)
    return fix_phase(U[:, :r])


def balanced_shape(n_samples, order):
    """Near-square mode sizes with sum n_samples + order - 1 (expfit.py:274-280)."""
    base, rem = divmod(n_samples + order - 1, order)
    return tuple([base + 1] * rem + [base] * (order - rem))
