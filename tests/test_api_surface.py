"""Drop-in check (CPU, no GPU calls): every public class/function of the
reference package on the product path exists here with the same parameter
names, and every public member of its classes exists too.  Needs the
reference checkout (this build container); skipped where it is absent (the
GPU box never has it)."""

import inspect
import os
import sys

import pytest

import paper_1401_6238_b200 as O

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference checkout absent")

# The hot path and its direct callers; the TLS /
# exponential-fitting / dense-builder functions are out of scope.
NAMES = ["AntiCirculantTensor", "BaabTensor", "BhhbTensor", "DENSE_CAP", "HankelTensor",
         "LevelKHankelTensor", "TuckerResult", "fft1", "fft2", "fftn", "fourier_matrix",
         "hooi_symmetric", "ifft1", "ifft2", "ifftn", "times_matrices", "vec", "unvec"]


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, REF)
    try:
        import hankelfft
        from hankelfft import block
    finally:
        sys.path.remove(REF)
    return hankelfft, block


def _params(f):
    return list(inspect.signature(f).parameters)


def test_public_names_and_signatures(ref):
    R, block = ref
    for name in NAMES:
        r = getattr(R, name, None) or getattr(block, name)
        o = getattr(O, name, None)
        assert o is not None, f"missing {name}"
        if inspect.isclass(r):
            assert _params(r) == _params(o), name
            missing = {k for k in dir(r) if not k.startswith("_")} - set(dir(o))
            assert not missing, f"{name} lacks {sorted(missing)}"
            for k in dir(r):
                if k.startswith("_"):
                    continue
                ra, oa = getattr(r, k), getattr(o, k)
                if inspect.isfunction(ra):
                    assert _params(ra) == _params(oa), f"{name}.{k}"
        elif callable(r):
            assert _params(r) == _params(o), name
        else:
            assert r == o, name
