"""Round-2 golden fixtures, produced by running the REFERENCE implementation.

    python oracle/gen_golden_r2.py

Same read-only aliased import as ``gen_golden.py``.  Writes to tests/golden/:

* ``cfg5_sweep50.npz`` -- the reference's cfg5 loop (times_matrices ->
  truncated_left_singular_vectors, decompose.py:35-41 / hankel.py:174-194)
  run for 50 sweeps from the shared U0 on signals 0 and 1 (SURVEY §8(d) cfg5:
  final-U projector at 1e-10).
* ``tm_large.npz`` -- reference ``times_matrices`` on tensors whose d_H exceeds
  one on-chip transform (two-level plans here): order 3 n=3000 r=3 with the
  same matrix twice (the HOOI shape) and with distinct matrices, and order 2
  (5000, 4000) r=2.
* ``hooi_small.npz`` -- reference ``hooi_symmetric`` (decompose.py:142-184) on
  small square Hankel and BHHB tensors, including the rank-deficient all-ones
  tensor (factors must stay orthonormal).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from gen_golden import OUT, load_reference, rand_vec  # noqa: E402
from paper_1401_6238_b200 import workloads  # noqa: E402


def cfg5_sweep50(ref):
    sig, U0, shape = workloads.cfg5(signals=2)
    n = shape[0]
    out = {}
    for s in range(2):
        H = ref.HankelTensor(shape, sig[s])
        U = U0
        for _ in range(50):
            T = ref.times_matrices(H, [np.conj(U)] * 2)
            U = ref.truncated_left_singular_vectors(T.reshape(n, -1), 5)
        out[f"U50_{s}"] = U
        out[f"T50_norm_{s}"] = np.linalg.norm(T)
    np.savez(os.path.join(OUT, "cfg5_sweep50.npz"), **out)


def tm_large(ref):
    h3, M, M2, h2, Mb = workloads.tm_large_inputs()
    H = ref.HankelTensor((3000, 3000, 3000), h3)
    H2 = ref.HankelTensor((5000, 4000), h2)
    np.savez(os.path.join(OUT, "tm_large.npz"), T3_same=ref.times_matrices(H, [M, M]),
             T3_mixed=ref.times_matrices(H, [M, M2]), T2=ref.times_matrices(H2, [Mb]))


def hooi_small(ref):
    rng = np.random.default_rng(4242)
    out = {}
    cases = []
    # rank-deficient: all-ones Hankel (rank-1 unfolding), rank 2
    cases.append(("ones", ref.HankelTensor((5, 5, 5), np.ones(13)), 2))
    cases.append(("rand", ref.HankelTensor((6, 6, 6), rand_vec(rng, 16)), 2))
    cases.append(("rand4", ref.HankelTensor((5, 5, 5, 5), rand_vec(rng, 17)), 3))
    Hb = rand_vec(rng, 4 * 7).reshape(4, 7)
    cases.append(("bhhb", ref.BhhbTensor(3, (2, 2, 2), (3, 3, 3), Hb), 2))
    for name, T, r in cases:
        res = ref.hooi_symmetric(T, r, max_iter=30)
        U = res.factor
        out[f"{name}_P"] = U @ U.conj().T
        out[f"{name}_U"] = U
        out[f"{name}_core"] = res.core
        out[f"{name}_fits"] = np.array(res.fits)
        out[f"{name}_meta"] = np.array([res.converged, res.n_iter, res.monotone], dtype=np.int64)
    out["bhhb_H"] = Hb
    out["rand_h"] = cases[1][1].h
    out["rand4_h"] = cases[2][1].h
    np.savez(os.path.join(OUT, "hooi_small.npz"), **out)


def main():
    ref = load_reference()
    tm_large(ref)
    hooi_small(ref)
    cfg5_sweep50(ref)
    print("round-2 golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
