"""Knot vectors and tensor spaces (host-side metadata mirroring splines.py).

Same names, validation rules and index conventions as the reference
(splines.py:16-96, 195-259); only lightweight host data lives here.  The
collocation matrices are produced natively by ``mfwq_rule1d_build``.
"""

from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class KnotVector:
    """Open knot vector of degree ``degree`` on [0, 1] (splines.py:16-49)."""

    degree: int
    knots: np.ndarray = field(repr=False)

    def __post_init__(self):
        p = self.degree
        if p < 1:
            raise ValueError(f"degree must be >= 1, got {p}")
        t = np.ascontiguousarray(np.asarray(self.knots, dtype=float))
        t.setflags(write=False)
        object.__setattr__(self, "knots", t)
        if t.ndim != 1 or len(t) < 2 * (p + 1):
            raise ValueError("knot vector too short for the given degree")
        if np.any(np.diff(t) < 0):
            raise ValueError("knots must be nondecreasing")
        if t[0] != 0.0 or t[-1] != 1.0:
            raise ValueError("knot vector must start at 0 and end at 1")
        if np.any(t[: p + 1] != 0.0) or np.any(t[-(p + 1):] != 1.0):
            raise ValueError("knot vector must be open (p+1 repeats at each end)")
        if t[p + 1] == 0.0 or t[-(p + 2)] == 1.0:
            raise ValueError("endpoint multiplicity must be exactly p+1")
        inner = t[p + 1: len(t) - p - 1]
        if len(inner) and np.unique(inner, return_counts=True)[1].max() > p:
            raise ValueError("interior knot multiplicity exceeds p")

    @property
    def n_funcs(self) -> int:
        return len(self.knots) - self.degree - 1

    @property
    def n_interior(self) -> int:
        return self.n_funcs - 2

    @property
    def breakpoints(self) -> np.ndarray:
        return np.unique(self.knots)

    @property
    def n_elements(self) -> int:
        return len(self.breakpoints) - 1

    def support(self, i: int):
        return float(self.knots[i]), float(self.knots[i + self.degree + 1])


def make_uniform_knots(p: int, n_el: int) -> KnotVector:
    """splines.py:88-96."""
    if p < 1:
        raise ValueError(f"degree must be >= 1, got {p}")
    if n_el < 1:
        raise ValueError(f"number of elements must be >= 1, got {n_el}")
    return KnotVector(p, np.concatenate([np.zeros(p + 1), np.arange(1, n_el) / n_el, np.ones(p + 1)]))


@dataclass(frozen=True)
class TensorSpace:
    """Tensor product space with Dirichlet boundary removal (splines.py:195-223)."""

    knotvectors: tuple

    def __post_init__(self):
        object.__setattr__(self, "knotvectors", tuple(self.knotvectors))
        for kv in self.knotvectors:
            if kv.n_funcs - 2 < 1:
                raise ValueError("each direction needs at least one interior function")

    @property
    def dim(self) -> int:
        return len(self.knotvectors)

    @property
    def n_per_dir(self):
        return tuple(kv.n_funcs - 2 for kv in self.knotvectors)

    @property
    def n_dofs(self) -> int:
        return int(np.prod(self.n_per_dir))


def tensor_space(p: int, n_el: int, d: int = 3) -> TensorSpace:
    """splines.py:226-229."""
    kv = make_uniform_knots(p, n_el)
    return TensorSpace((kv,) * d)


def multi_to_scalar(multi, dims) -> int:
    """1-based multi-index -> 1-based scalar, direction 1 fastest (splines.py:232-246)."""
    multi = tuple(int(i) for i in multi)
    dims = tuple(int(s) for s in dims)
    if len(multi) != len(dims):
        raise ValueError("multi-index and dims length mismatch")
    out, stride = 1, 1
    for i, s in zip(multi, dims):
        if not 1 <= i <= s:
            raise ValueError(f"index component {i} out of range 1..{s}")
        out += (i - 1) * stride
        stride *= s
    return out


def scalar_to_multi(i: int, dims):
    """Inverse of multi_to_scalar (splines.py:249-259)."""
    dims = tuple(int(s) for s in dims)
    if not 1 <= i <= int(np.prod(dims)):
        raise ValueError(f"scalar index {i} out of range")
    rem, out = i - 1, []
    for s in dims:
        out.append(rem % s + 1)
        rem //= s
    return tuple(out)
