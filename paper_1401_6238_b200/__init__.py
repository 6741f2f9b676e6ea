"""B200-native fast Hankel tensor-vector products (arXiv 1401.6238).

Drop-in for the hot path of the reference package ``hankelfft`` 0.1.0: the
same classes and functions as ``hankelfft.hankel`` and ``hankelfft.block``
(re-exported by the reference ``__init__.py:4-43``), with every product
computed by hand-written sm_100a CUDA kernels behind the C ABI in
``include/hankelfft_b200.h``.  ``batched`` exposes the device-level batched
engine on torch CUDA tensors.

    import paper_1401_6238_b200 as hankelfft
    y = hankelfft.HankelTensor(shape, h).tvp_partial([x, x])
"""

from .block import BaabTensor, BhhbTensor, LevelKHankelTensor, unvec, vec
from .fourier import fft1, fft2, fftn, fourier_matrix, ifft1, ifft2, ifftn
from .hankel import DENSE_CAP, AntiCirculantTensor, HankelTensor, times_matrices
from .hooi import TuckerResult, hooi_symmetric

__version__ = "0.1.0"

__all__ = [
    "AntiCirculantTensor",
    "BaabTensor",
    "BhhbTensor",
    "DENSE_CAP",
    "HankelTensor",
    "LevelKHankelTensor",
    "TuckerResult",
    "fft1",
    "fft2",
    "fftn",
    "fourier_matrix",
    "hooi_symmetric",
    "ifft1",
    "ifft2",
    "ifftn",
    "times_matrices",
    "unvec",
    "vec",
]
