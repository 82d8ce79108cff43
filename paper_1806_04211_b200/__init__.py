"""B200-native block-tiled Gaussian elimination over GF(p) (arXiv 1806.04211).

Drop-in for the reference ``gfrref`` block-elimination path: ChopMatrix,
the ClearDown/ECH, Extend, UpdateRow/UpdateRowTrafo and clean-up jobs and
the ``echelonize`` entry point, computed by hand-written sm_100a kernels
(``csrc/``) behind the C ABI in ``include/gfq.h``.  ``gfrref`` mirrors the
reference API in Python over that ABI.
"""
from . import gfrref  # noqa: F401
from .gfrref import (  # noqa: F401
    BitString, ChopSpec, EchelonizeOptions, EchelonOutput, EchResult, FieldSpec, IndexSet, Matrix, PkgA, PkgD,
    PkgE, adi, cex, chop, clear_down, clear_up, copy_d, crz, ech, echelonize, extend, mad, mat_build, mkr, mul,
    pre_clear_up, random_matrix, random_product_matrix, rex, row_lengthen, rrf, un0, unh, update_row,
    update_row_trafo)
