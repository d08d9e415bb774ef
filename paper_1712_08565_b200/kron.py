"""Cost meter, tensor-grid ordering and a device Kronecker apply (mirrors kron.py)."""

import ctypes as C

import numpy as np
import scipy.sparse as sp

from . import _dev, _lib


class CostMeter:
    """Flop / scratch accounting with the reference's conventions (kron.py:14-33)."""

    def __init__(self):
        self.flops = 0
        self.bytes_peak = 0

    def add_flops(self, n: int):
        self.flops += int(n)

    def note_buffers(self, n_scalars: int):
        self.bytes_peak = max(self.bytes_peak, int(n_scalars))

    def reset(self):
        self.flops = 0
        self.bytes_peak = 0


def tensor_grid(points_per_dir):
    """Flat coordinate arrays, direction 1 fastest (kron.py:136-145)."""
    rev = np.meshgrid(*reversed([np.asarray(q) for q in points_per_dir]), indexing="ij")
    return [g.ravel() for g in reversed(rev)]


def kron_apply(factors, x, meter: CostMeter | None = None, accumulate_into=None):
    """(A_d x ... x A_1) x on the GPU, direction d first (kron.py:70-100).

    ``x`` may be a numpy array (result returned as numpy) or a CUDA tensor.
    """
    d = len(factors)
    dense = [np.ascontiguousarray(f.toarray() if sp.issparse(f) else np.asarray(f, dtype=float)) for f in factors]
    rows = np.array([f.shape[0] for f in dense], dtype=np.int32)
    cols = np.array([f.shape[1] for f in dense], dtype=np.int32)
    xt, host = _dev.to_device(x)
    if xt.numel() != int(np.prod(cols)):
        raise ValueError(f"vector length {xt.numel()} does not match operator columns {int(np.prod(cols))}")
    y = accumulate_into if accumulate_into is not None else _dev.empty(int(np.prod(rows)))
    ptrs = (_lib.dp * d)(*[_lib.dptr(f) for f in dense])
    _lib.check(_lib.lib().mfwq_kron_apply(d, _lib.iptr(rows), _lib.iptr(cols), ptrs, C.c_void_p(xt.data_ptr()),
                                          C.c_void_p(y.data_ptr()), 1 if accumulate_into is not None else 0,
                                          C.c_void_p(_dev.stream_ptr())))
    if meter is not None:
        t = list(cols)
        for l in range(d - 1, -1, -1):
            ncols = int(np.prod([t[k] for k in range(d) if k != l]))
            A = factors[l]
            meter.add_flops(2 * (A.nnz if sp.issparse(A) else A.shape[0] * A.shape[1]) * ncols)
            t[l] = rows[l]
    return _dev.back(y, host)
