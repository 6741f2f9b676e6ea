"""CPU-side checks of the C ABI: the library loads and exports every entry
point declared in include/hankelfft_b200.h; host-side validation paths that
do not need a GPU."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_1401_6238_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hankelfft_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hk_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_expected_api():
    names = declared_functions()
    for must in ["hk_plan_create_hankel", "hk_tvp_partial", "hk_tvp_full", "hk_spectrum",
                 "hk_times_matrices", "hk_last_error"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = N.load_library()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert set(declared_functions()) == set(N.EXPORTED)


def test_version_and_error_string_without_gpu():
    lib = N.load_library()
    assert lib.hk_version() >= 100
    # a NULL plan is rejected before touching CUDA
    rc = lib.hk_tvp_partial(None, N.Operand(0, 0, 0, 0), None, 0, 1, None, 0, None, None)
    assert rc == N.HK_EINVAL
    assert b"plan" in lib.hk_last_error()


def test_plan_rejects_bad_shapes_without_gpu():
    lib = N.load_library()
    h = ctypes.c_void_p()
    rc = lib.hk_plan_create_hankel(ctypes.byref(h), 1, N.i64_array([3]), 0)
    assert rc == N.HK_EINVAL and b"order must be at least 2" in lib.hk_last_error()
    rc = lib.hk_plan_create_hankel(ctypes.byref(h), 3, N.i64_array([3, 0, 2]), 0)
    assert rc == N.HK_EINVAL and b"positive" in lib.hk_last_error()
    rc = lib.hk_plan_create_hankel(ctypes.byref(h), 3, N.i64_array([3, 3, 3]), 4)
    assert rc == N.HK_EINVAL and b"shorter than d_H" in lib.hk_last_error()


def test_python_validation_matches_reference_messages():
    import paper_1401_6238_b200 as P

    with pytest.raises(ValueError, match="generating vector must have length 7, got 6"):
        P.HankelTensor((3, 3, 3), np.zeros(6))
    with pytest.raises(ValueError, match="shape entries must be positive"):
        P.HankelTensor((3, 0), np.zeros(2))
    H = P.HankelTensor((3, 3, 3), np.zeros(7))
    with pytest.raises(ValueError, match="expected 2 vectors, got 1"):
        H.tvp_partial([np.zeros(3)])
    with pytest.raises(ValueError, match="mode-2 vector must have length 3"):
        H.tvp_partial([np.zeros(3), np.zeros(4)])
    with pytest.raises(ValueError, match="order must be at least 2"):
        P.AntiCirculantTensor(1, 3, np.zeros(3))
    with pytest.raises(ValueError, match="compressed generating vector must have length 4"):
        P.AntiCirculantTensor(3, 4, np.zeros(3))
    with pytest.raises(ValueError, match="generating matrix must be 4x4"):
        P.BhhbTensor(3, (2, 2, 2), (2, 2, 2), np.zeros((4, 5)))
    with pytest.raises(ValueError, match="vector must have length 4"):
        P.unvec(np.zeros(3), 2, 2)
    with pytest.raises(ValueError, match="expected 2 matrices, got 1"):
        P.times_matrices(H, [np.eye(3)])
    with pytest.raises(ValueError, match="matrix 1 must have 3 rows"):
        P.times_matrices(H, [np.eye(3), np.eye(4)])


def test_structural_helpers_without_gpu():
    import paper_1401_6238_b200 as P
    from oracle import hankel_oracle as O

    H = P.HankelTensor((3, 3, 3), np.arange(7))
    np.testing.assert_array_equal(H.reduced_unfold(0).real,
                                  [[0, 1, 2, 3, 4], [1, 2, 3, 4, 5], [2, 3, 4, 5, 6]])
    assert H.embed().dim == 7 and H.is_square and H.dof == 7
    np.testing.assert_array_equal(H.to_dense(), O.dense_hankel(np.arange(7), (3, 3, 3)))
    rng = np.random.default_rng(0)
    G = rng.standard_normal((4, 3, 3))
    L = P.LevelKHankelTensor(2, ((2, 3), (2, 2), (2, 2)), G)
    np.testing.assert_array_equal(L.to_dense(),
                                  O.dense_level_k(G, ((2, 3), (2, 2), (2, 2))))
    B = P.BhhbTensor(3, (2, 3, 2), (3, 2, 2), rng.standard_normal((5, 5)))
    np.testing.assert_array_equal(B.to_dense(), O.dense_bhhb(B.H, B.block_shape, B.outer_shape))
    pairs = P.AntiCirculantTensor(3, 3, [1, 2, 3]).special_eigenpairs()
    assert pairs[0][0] == pytest.approx(18.0)


def test_fourier_wrappers_validate_without_gpu():
    import paper_1401_6238_b200 as P

    with pytest.raises(ValueError, match="empty input"):
        P.fft1(np.array([]))
    with pytest.raises(ValueError, match="size must be positive"):
        P.fourier_matrix(0)
    np.testing.assert_allclose(P.fourier_matrix(2), [[1, 1], [1, -1]], atol=1e-15)
