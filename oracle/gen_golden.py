"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python oracle/gen_golden.py            # all fixtures
    python oracle/gen_golden.py --skip-cfg3  # skip the ~25 s cfg3 product

The reference package is imported read-only under the alias ``hankelfft_ref``
from ``/root/reference/pkg/src/hankelfft`` (parity-harness tip).
Outputs go to ``tests/golden/``; they are committed, so the GPU box (which has
no /root/reference) can check both the oracle and the CUDA path against the
reference's own numbers.
"""

from __future__ import annotations

import argparse
import importlib.util
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF_PKG = "/root/reference/pkg/src/hankelfft"
OUT = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)

from paper_1401_6238_b200 import workloads  # noqa: E402


def load_reference():
    spec = importlib.util.spec_from_file_location(
        "hankelfft_ref", os.path.join(REF_PKG, "__init__.py"),
        submodule_search_locations=[REF_PKG])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["hankelfft_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def rand_vec(rng, n):
    return rng.standard_normal(n) + 1j * rng.standard_normal(n)


def small_cases(ref):
    """Random small products of every structured type, reference outputs."""
    rng = np.random.default_rng(20260101)
    out = {}
    # Hankel, orders 2..5, square and non-square, dims 1..9 (incl. order-2 matrices)
    hk = []
    for i in range(120):
        m = int(rng.integers(2, 6))
        shape = tuple(int(rng.integers(1, 10)) for _ in range(m))
        d = sum(shape) - m + 1
        h = rand_vec(rng, d)
        xs = [rand_vec(rng, n) for n in shape]
        H = ref.HankelTensor(shape, h)
        hk.append((shape, h, xs, H.tvp_partial(xs[1:]), H.tvp_full(xs)))
    out["hankel"] = hk
    ac = []
    for i in range(40):
        m = int(rng.integers(2, 5))
        n = int(rng.integers(1, 12))
        c = rand_vec(rng, n)
        xs = [rand_vec(rng, n) for _ in range(m)]
        A = ref.AntiCirculantTensor(m, n, c)
        ac.append((m, c, xs, A.spectrum, A.tvp_partial(xs[1:]), A.tvp_full(xs)))
    out["acirc"] = ac
    bh = []
    for i in range(40):
        m = int(rng.integers(2, 4))
        block = tuple(int(rng.integers(1, 6)) for _ in range(m))
        outer = tuple(int(rng.integers(1, 5)) for _ in range(m))
        din, dout = sum(block) - m + 1, sum(outer) - m + 1
        Hm = rand_vec(rng, din * dout).reshape(din, dout)
        xs = [rand_vec(rng, b * o) for b, o in zip(block, outer)]
        T = ref.BhhbTensor(m, block, outer, Hm)
        bh.append((block, outer, Hm, xs, T.tvp_partial(xs[1:]), T.tvp_full(xs)))
    out["bhhb"] = bh
    ba = []
    for i in range(30):
        m = int(rng.integers(2, 4))
        n, N = int(rng.integers(1, 6)), int(rng.integers(1, 5))
        C = rand_vec(rng, n * N).reshape(n, N)
        xs = [rand_vec(rng, n * N) for _ in range(m)]
        T = ref.BaabTensor(m, C)
        ba.append((m, C, xs, T.tvp_partial(xs[1:]), T.tvp_full(xs)))
    out["baab"] = ba
    lk = []
    for i in range(30):
        m = int(rng.integers(2, 4))
        k = int(rng.integers(1, 4))
        levels = tuple(tuple(int(rng.integers(1, 4)) for _ in range(m)) for _ in range(k))
        gshape = tuple(sum(lv) - m + 1 for lv in levels)
        G = rand_vec(rng, int(np.prod(gshape))).reshape(gshape)
        sizes = [int(np.prod([lv[p] for lv in levels])) for p in range(m)]
        xs = [rand_vec(rng, s) for s in sizes]
        T = ref.LevelKHankelTensor(m, levels, G)
        lk.append((levels, G, xs, T.tvp_partial(xs[1:]), T.tvp_full(xs)))
    out["levelk"] = lk
    tm = []
    for i in range(20):
        m = int(rng.integers(2, 5))
        shape = tuple(int(rng.integers(1, 8)) for _ in range(m))
        d = sum(shape) - m + 1
        h = rand_vec(rng, d)
        mats = [rand_vec(rng, n * r).reshape(n, r)
                for n, r in zip(shape[1:], rng.integers(1, 4, m - 1))]
        H = ref.HankelTensor(shape, h)
        tm.append((shape, h, mats, ref.times_matrices(H, mats)))
    out["times_matrices"] = tm
    return out


def save_pickled(name, obj):
    np.save(os.path.join(OUT, name), np.array(obj, dtype=object), allow_pickle=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-cfg3", action="store_true")
    args = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    ref = load_reference()

    save_pickled("small_cases.npy", small_cases(ref))

    # cfg1: full inputs and outputs + dense 100^3 contraction
    h, x = workloads.cfg1()
    H = ref.HankelTensor((100,) * 3, h)
    dense = ref.core.dense_hankel(h, (100,) * 3)
    np.savez(os.path.join(OUT, "cfg1.npz"),
             y=H.tvp_partial([x, x]), alpha=np.array(H.tvp_full([x, x, x])),
             y_dense=ref.core.tvp_partial(dense, [x, x]),
             alpha_dense=np.array(ref.core.tvp_full(dense, [x, x, x])))

    # cfg2: reference exact-L outputs for a few products + per-product norms
    hb, xb = workloads.cfg2()
    sel = np.array([0, 1, 2, 4095])
    ys = []
    norms = np.empty(hb.shape[0])
    first = np.empty(hb.shape[0], dtype=np.complex128)
    for b in range(hb.shape[0]):
        y = ref.HankelTensor((1024,) * 4, hb[b]).tvp_partial([xb[b]] * 3)
        norms[b] = np.linalg.norm(y)
        first[b] = y[0]
        if b in sel:
            ys.append(y)
    np.savez(os.path.join(OUT, "cfg2.npz"), sel=sel, y=np.array(ys), norms=norms, first=first,
             h_sum=hb.sum(axis=1)[:8], x_sum=xb.sum(axis=1)[:8])

    # cfg4: BHHB outputs for two products + norms of all
    Hb, Xb = workloads.cfg4()
    sel4 = np.array([0, 1023])
    ys4 = []
    norms4 = np.empty(Hb.shape[0])
    for b in range(Hb.shape[0]):
        xv = Xb[b].ravel(order="F")
        y = ref.BhhbTensor(3, (64,) * 3, (64,) * 3, Hb[b]).tvp_partial([xv, xv])
        norms4[b] = np.linalg.norm(y)
        if b in sel4:
            ys4.append(y)
    np.savez(os.path.join(OUT, "cfg4.npz"), sel=sel4, y=np.array(ys4), norms=norms4)

    # cfg5: signal 0, two HOOI iterations from U0 via the reference
    sig, U0, shape = workloads.cfg5(signals=2)
    Hs = ref.HankelTensor(shape, sig[0])
    T1 = ref.times_matrices(Hs, [np.conj(U0)] * 2)
    U1 = ref.truncated_left_singular_vectors(T1.reshape(shape[0], -1), 5)
    T2 = ref.times_matrices(Hs, [np.conj(U1)] * 2)
    U2 = ref.truncated_left_singular_vectors(T2.reshape(shape[0], -1), 5)
    rows = np.arange(0, shape[0], 10)
    np.savez(os.path.join(OUT, "cfg5.npz"), rows=rows, T1_rows=T1[rows], T2_rows=T2[rows],
             T1_norm=np.linalg.norm(T1), T2_norm=np.linalg.norm(T2), U1=U1, U2=U2,
             sig0_sum=sig[0].sum(), U0=U0)

    if not args.skip_cfg3:
        h3, x3 = workloads.cfg3()
        y3 = ref.HankelTensor((1 << 22,) * 3, h3).tvp_partial([x3, x3])
        rng = np.random.default_rng(33)
        idx = np.sort(rng.choice(1 << 22, 4096, replace=False))
        idx[0] = 0
        idx[-1] = (1 << 22) - 1
        np.savez(os.path.join(OUT, "cfg3.npz"), idx=idx, y=y3[idx], norm=np.linalg.norm(y3),
                 ysum=y3.sum())
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
