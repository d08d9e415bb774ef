"""Host-side spline metadata: open knot vectors on [0, 1] and tensor spaces.

The B200 path only needs sizes, breakpoints and the flat index convention on
the host (the collocation tables themselves come from ``mfwq_rule1d_build``).
The public names, the ValueError conditions and their messages, and the index
maps are those of the reference (splines.py:16-96, 195-259), so callers and
the reference's own tests see the same behaviour.
"""

from dataclasses import dataclass, field

import numpy as np


def _knot_errors(p: int, t: np.ndarray):
    """Yield the first violated rule of an open knot vector (splines.py:26-49 semantics)."""
    yield t.ndim != 1 or t.size < 2 * p + 2, "knot vector too short for the given degree"
    yield bool((t[1:] < t[:-1]).any()), "knots must be nondecreasing"
    yield t[0] != 0.0 or t[-1] != 1.0, "knot vector must start at 0 and end at 1"
    ends = np.concatenate([t[: p + 1], 1.0 - t[t.size - p - 1:]])
    yield bool(ends.any()), "knot vector must be open (p+1 repeats at each end)"
    yield t[p + 1] == 0.0 or t[t.size - p - 2] == 1.0, "endpoint multiplicity must be exactly p+1"
    mid = t[p + 1: t.size - p - 1]
    yield mid.size > 0 and np.unique(mid, return_counts=True)[1].max() > p, \
        "interior knot multiplicity exceeds p"


@dataclass(frozen=True)
class KnotVector:
    """Open knot vector: ``degree`` p, p+1 repeated end knots, interior multiplicity <= p."""

    degree: int
    knots: np.ndarray = field(repr=False)

    def __post_init__(self):
        if self.degree < 1:
            raise ValueError(f"degree must be >= 1, got {self.degree}")
        t = np.array(self.knots, dtype=np.float64, copy=True).reshape(-1) \
            if np.ndim(self.knots) == 1 else np.asarray(self.knots, dtype=np.float64)
        t.setflags(write=False)
        object.__setattr__(self, "knots", t)
        for bad, msg in _knot_errors(self.degree, t):
            if bad:
                raise ValueError(msg)

    # sizes: n_funcs basis functions on the full space, two of them removed by the Dirichlet BC
    @property
    def n_funcs(self) -> int:
        return self.knots.size - (self.degree + 1)

    @property
    def n_interior(self) -> int:
        return self.n_funcs - 2

    @property
    def breakpoints(self) -> np.ndarray:
        return np.unique(self.knots)

    @property
    def n_elements(self) -> int:
        return self.breakpoints.size - 1

    def support(self, i: int):
        """Closed support [t_i, t_{i+p+1}] of basis function i (0-based)."""
        return float(self.knots[i]), float(self.knots[i + self.degree + 1])


def make_uniform_knots(p: int, n_el: int) -> KnotVector:
    """Uniform open knot vector with n_el spans (splines.py:88-96)."""
    for name, v in (("degree", p), ("number of elements", n_el)):
        if v < 1:
            raise ValueError(f"{name} must be >= 1, got {v}")
    t = np.zeros(n_el + 2 * p + 1)
    t[p + 1: p + n_el] = np.arange(1, n_el) / n_el
    t[p + n_el:] = 1.0
    return KnotVector(p, t)


@dataclass(frozen=True)
class TensorSpace:
    """Tensor-product space of the given knot vectors, Dirichlet functions removed."""

    knotvectors: tuple

    def __post_init__(self):
        kvs = tuple(self.knotvectors)
        object.__setattr__(self, "knotvectors", kvs)
        if any(kv.n_interior < 1 for kv in kvs):
            raise ValueError("each direction needs at least one interior function")

    @property
    def dim(self) -> int:
        return len(self.knotvectors)

    @property
    def n_per_dir(self):
        return tuple(kv.n_interior for kv in self.knotvectors)

    @property
    def n_dofs(self) -> int:
        return int(np.prod(self.n_per_dir))


def tensor_space(p: int, n_el: int, d: int = 3) -> TensorSpace:
    """The same uniform knot vector in each of d directions (splines.py:226-229)."""
    return TensorSpace(tuple([make_uniform_knots(p, n_el)] * d))


def multi_to_scalar(multi, dims) -> int:
    """1-based multi-index -> 1-based flat index, direction 1 fastest (splines.py:232-246)."""
    idx = [int(i) for i in multi]
    ext = [int(s) for s in dims]
    if len(idx) != len(ext):
        raise ValueError("multi-index and dims length mismatch")
    for i, s in zip(idx, ext):
        if i < 1 or i > s:
            raise ValueError(f"index component {i} out of range 1..{s}")
    strides = np.concatenate([[1], np.cumprod(ext[:-1])]).astype(np.int64)
    return 1 + int(np.dot(np.array(idx) - 1, strides))


def scalar_to_multi(i: int, dims):
    """Inverse of multi_to_scalar (splines.py:249-259)."""
    ext = [int(s) for s in dims]
    if i < 1 or i > int(np.prod(ext)):
        raise ValueError(f"scalar index {i} out of range")
    return tuple(int(v) + 1 for v in np.unravel_index(i - 1, ext, order="F"))
