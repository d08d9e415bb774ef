"""Geometry maps (mirrors geometry.py names).

Analytic maps carry a ``kind`` the device coefficient kernel understands
(identity, the analytic quarter ring, affine); their Jacobians are then
evaluated on the GPU at every quadrature point.  Any other object with
``jacobian(xi)`` (for instance the reference's own rational or spline maps)
is evaluated on the host once at setup and uploaded (MFWQ_GEOM_JACOBIAN).
"""

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np


@dataclass(frozen=True)
class GeometryMap:
    dim: int
    kind: str
    _map: Callable
    _jacobian: Callable
    A: Optional[np.ndarray] = None
    b: Optional[np.ndarray] = None

    def evaluate(self, xi):
        return self._map(np.atleast_2d(np.asarray(xi, dtype=float)))

    def jacobian(self, xi):
        return self._jacobian(np.atleast_2d(np.asarray(xi, dtype=float)))


def identity_map(d: int = 3) -> GeometryMap:
    """geometry.py:47-54."""
    return GeometryMap(d, "identity", lambda xi: xi.copy(),
                       lambda xi: np.broadcast_to(np.eye(d), (len(xi), d, d)).copy())


def affine_map(A, b) -> GeometryMap:
    """geometry.py:57-70."""
    A = np.asarray(A, dtype=float)
    b = np.asarray(b, dtype=float)
    d = A.shape[0]
    if np.linalg.det(A) <= 0:
        raise ValueError("affine map must be orientation-preserving")
    return GeometryMap(d, "affine", lambda xi: xi @ A.T + b,
                       lambda xi: np.broadcast_to(A, (len(xi), d, d)).copy(), A=A, b=b)


def quarter_ring_map() -> GeometryMap:
    """Analytic thick quarter ring (geometry.py:73-96)."""

    def _map(xi):
        r = 1.0 + xi[:, 0]
        th = np.pi / 2 * xi[:, 1]
        return np.stack([r * np.cos(th), r * np.sin(th), xi[:, 2]], axis=1)

    def _jac(xi):
        r = 1.0 + xi[:, 0]
        th = np.pi / 2 * xi[:, 1]
        c, s = np.cos(th), np.sin(th)
        J = np.zeros((len(xi), 3, 3))
        J[:, 0, 0] = c
        J[:, 0, 1] = -np.pi / 2 * r * s
        J[:, 1, 0] = s
        J[:, 1, 1] = np.pi / 2 * r * c
        J[:, 2, 2] = 1.0
        return J

    return GeometryMap(3, "analytic-quarter-ring", _map, _jac)


def device_kind(geom):
    """(kind code, affine matrix) for maps the coefficient kernel evaluates itself."""
    kind = getattr(geom, "kind", None)
    if kind == "identity":
        return 0, None
    if kind == "analytic-quarter-ring":
        return 1, None
    if kind == "affine":
        A = getattr(geom, "A", None)
        if A is None:  # the reference's affine_map: J is constant, read it once
            A = np.asarray(geom.jacobian(np.zeros((1, 3))))[0]
        return 2, np.ascontiguousarray(A, dtype=float)
    return 3, None
