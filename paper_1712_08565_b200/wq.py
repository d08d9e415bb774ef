"""Weighted-quadrature rules, built natively (mirrors wq.py names).

``build_wq_rule`` calls ``mfwq_rule1d_build`` (C++: Cox-de Boor
collocation, exact Gram by Gauss-Legendre, per-row min-norm least squares
with numpy's truncation rule, boundary-point retry) and wraps the result in
the same object shape as the reference (wq.py:126-205): ``points``,
``weights[(a, b)]`` (n_funcs x n_points CSR) and ``colloc[b]``
(n_points x n_funcs CSR).
"""

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from . import _lib
from .errors import WQConstructionError  # noqa: F401  (re-export)

EXACTNESS_TOL = 1e-10
_PAIRS = ((0, 0), (0, 1), (1, 0), (1, 1))


@dataclass(frozen=True)
class WQRule1D:
    kv: object
    points: np.ndarray = field(repr=False)
    weights: dict = field(repr=False)
    colloc: dict = field(repr=False)
    boundary_extra: int = 0

    @property
    def n_points(self) -> int:
        return len(self.points)


def build_wq_rule(kv) -> WQRule1D:
    L = _lib.lib()
    knots = np.ascontiguousarray(kv.knots, dtype=float)
    h = C.c_void_p()
    _lib.check(L.mfwq_rule1d_build(int(kv.degree), len(knots), _lib.dptr(knots), C.byref(h)))
    try:
        npts, nfun, extra = C.c_int(), C.c_int(), C.c_int()
        nnz = np.zeros(6, dtype=np.int32)
        _lib.check(L.mfwq_rule1d_sizes(h, C.byref(npts), C.byref(nfun), C.byref(extra), _lib.iptr(nnz)))
        m, n = npts.value, nfun.value
        pts = np.empty(m)
        rows = [n] * 4 + [m] * 2
        cols = [m] * 4 + [n] * 2
        indptr = [np.empty(r + 1, dtype=np.int32) for r in rows]
        indices = [np.empty(max(int(z), 1), dtype=np.int32) for z in nnz]
        data = [np.empty(max(int(z), 1)) for z in nnz]
        _lib.check(L.mfwq_rule1d_export(
            h, _lib.dptr(pts), (_lib.ip * 6)(*[_lib.iptr(a) for a in indptr]),
            (_lib.ip * 6)(*[_lib.iptr(a) for a in indices]), (_lib.dp * 6)(*[_lib.dptr(a) for a in data])))
    finally:
        L.mfwq_rule1d_destroy(h)
    mats = [sp.csr_matrix((data[k][: nnz[k]], indices[k][: nnz[k]], indptr[k]), shape=(rows[k], cols[k]))
            for k in range(6)]
    pts.setflags(write=False)
    return WQRule1D(kv=kv, points=pts, weights={ab: mats[k] for k, ab in enumerate(_PAIRS)},
                    colloc={0: mats[4], 1: mats[5]}, boundary_extra=extra.value)


@dataclass(frozen=True)
class TensorRule:
    """Per-direction rules seen as one tensor rule (wq.py:167-205)."""

    rules: tuple

    def __post_init__(self):
        object.__setattr__(self, "rules", tuple(self.rules))

    @property
    def dim(self) -> int:
        return len(self.rules)

    @property
    def n_points_per_dir(self):
        return tuple(r.n_points for r in self.rules)

    @property
    def n_points(self) -> int:
        return int(np.prod(self.n_points_per_dir))

    def point_arrays(self):
        from .kron import tensor_grid
        return tensor_grid([r.points for r in self.rules])


def build_tensor_rule(space) -> TensorRule:
    """wq.py:208-210; identical directions are built once."""
    cache = {}
    rules = []
    for kv in space.knotvectors:
        key = (int(kv.degree), np.asarray(kv.knots, dtype=float).tobytes())
        if key not in cache:
            cache[key] = build_wq_rule(kv)
        rules.append(cache[key])
    return TensorRule(tuple(rules))
