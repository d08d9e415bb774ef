"""Load vector and error norms on the device (mirrors problems.py / assembly.py).

``assemble_rhs(space, geom, f)``                 assembly.py:201-230
``l2_relative_error(space, geom, u, case)``      problems.py:153-158
``h1_relative_error(space, geom, u, case)``      problems.py:145-150
``cube_sine_case()`` / ``oscillating_case()``    problems.py:77-94

The tensor-Gauss integrals run in ``csrc/quadrature.cu`` (sum-factorised over element blocks,
through ``mfwq_quad_*`` in include/mfwq.h).  The two built-in manufactured cases are evaluated in
the kernel at the mapped Gauss points (closed forms of the reference's sympy derivation).  Any
other integrand -- a host callable ``f(x)`` or a case object with ``u`` / ``grad_u`` callables,
for instance the reference's own ``ManufacturedCase`` -- is evaluated once on the host at the mapped
Gauss points and handed to the same kernels; the quadrature itself always runs on the GPU.
"""

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _dev, _lib
from .geometry import device_kind

CASE_VALUES, CASE_CUBE_SINE, CASE_RING_OSC = 0, 1, 2


@dataclass(frozen=True)
class ManufacturedCase:
    """Exact solution, gradient and matching source term (physical coordinates), problems.py:38-48."""

    name: str
    u: callable = field(repr=False)
    grad_u: callable = field(repr=False)
    f: callable = field(repr=False)
    alpha: float = 0.0
    reference_h1_errors: dict = field(default_factory=dict, repr=False)
    device_case: int = CASE_VALUES  # built-in device integrand, 0 = none


def _tag(fn, case_id):
    fn._mfwq_case = case_id
    return fn


def cube_sine_case() -> ManufacturedCase:
    """u = sin(pi x) sin(pi y) sin(pi z) on the unit cube, f = -lap u (problems.py:89-94)."""

    def u(x):
        x = np.atleast_2d(x)
        return np.sin(np.pi * x[:, 0]) * np.sin(np.pi * x[:, 1]) * np.sin(np.pi * x[:, 2])

    def grad_u(x):
        x = np.atleast_2d(x)
        s, c = np.sin(np.pi * x), np.cos(np.pi * x)
        return np.pi * np.stack([c[:, 0] * s[:, 1] * s[:, 2], s[:, 0] * c[:, 1] * s[:, 2],
                                 s[:, 0] * s[:, 1] * c[:, 2]], axis=1)

    def f(x):
        return 3.0 * np.pi ** 2 * u(x)

    return ManufacturedCase("cube-sine", _tag(u, CASE_CUBE_SINE), _tag(grad_u, CASE_CUBE_SINE),
                            _tag(f, CASE_CUBE_SINE), 0.0, {}, CASE_CUBE_SINE)


def oscillating_case() -> ManufacturedCase:
    """u = sin(5 pi x) sin(5 pi y) sin(5 pi z) (r^2 - 1)(r^2 - 4) on the quarter ring (problems.py:77-86)."""
    k = 5.0 * np.pi

    def parts(x):
        x = np.atleast_2d(x)
        s, c = np.sin(k * x), np.cos(k * x)
        S = s[:, 0] * s[:, 1] * s[:, 2]
        dS = k * np.stack([c[:, 0] * s[:, 1] * s[:, 2], s[:, 0] * c[:, 1] * s[:, 2], s[:, 0] * s[:, 1] * c[:, 2]], axis=1)
        r2 = x[:, 0] ** 2 + x[:, 1] ** 2
        h = (r2 - 1.0) * (r2 - 4.0)
        dh = np.stack([(4 * r2 - 10) * x[:, 0], (4 * r2 - 10) * x[:, 1], np.zeros(len(x))], axis=1)
        return S, dS, r2, h, dh

    def u(x):
        S, _, _, h, _ = parts(x)
        return S * h

    def grad_u(x):
        S, dS, _, h, dh = parts(x)
        return h[:, None] * dS + S[:, None] * dh

    def f(x):
        S, dS, r2, h, dh = parts(x)
        return -(h * (-3.0 * k * k * S) + 2.0 * np.sum(dS * dh, axis=1) + S * (16.0 * r2 - 20.0))

    return ManufacturedCase("quarter-ring-oscillating", _tag(u, CASE_RING_OSC), _tag(grad_u, CASE_RING_OSC),
                            _tag(f, CASE_RING_OSC), 0.0, {}, CASE_RING_OSC)


class _Quad:
    """Device Gauss rule + collocation tables of a space (mfwq_quad_create)."""

    def __init__(self, space, pts_per_span):
        _dev.require_cuda()
        if getattr(space, "dim", 3) != 3:
            raise NotImplementedError("device quadrature is three-dimensional")
        L = _lib.lib()
        kvs = space.knotvectors
        knots = [np.ascontiguousarray(kv.knots, dtype=float) for kv in kvs]
        p = np.array([kv.degree for kv in kvs], np.int32)
        nk = np.array([len(k) for k in knots], np.int32)
        kp = (_lib.dp * 3)(*[_lib.dptr(k) for k in knots])
        h = C.c_void_p()
        _lib.check(L.mfwq_quad_create(_lib.iptr(p), _lib.iptr(nk), kp, int(pts_per_span or 0), C.byref(h)))
        self._h = h
        ng = np.zeros(3, np.int32)
        npts, ndofs = C.c_longlong(), C.c_longlong()
        _lib.check(L.mfwq_quad_sizes(h, _lib.iptr(ng), C.byref(npts), C.byref(ndofs)))
        self.ng, self.npts, self.ndofs = tuple(int(v) for v in ng), npts.value, ndofs.value
        if self.ndofs != space.n_dofs:
            raise ValueError("quadrature and space disagree on the number of DoFs")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib.lib().mfwq_quad_destroy(h)
            self._h = None

    def points(self):
        """Parametric Gauss points (npts, 3), direction 1 fastest, and the 1D rules."""
        L = _lib.lib()
        xs, ws = [], []
        for l in range(3):
            x, w = np.zeros(self.ng[l]), np.zeros(self.ng[l])
            _lib.check(L.mfwq_quad_points(self._h, l, _lib.dptr(x), _lib.dptr(w)))
            xs.append(x)
            ws.append(w)
        g3, g2, g1 = np.meshgrid(xs[2], xs[1], xs[0], indexing="ij")
        return np.stack([g1.ravel(), g2.ravel(), g3.ravel()], axis=1), xs, ws


def _geometry_args(geom, quad):
    """(kind, affine12 host array, J device tensor or None) for the quadrature kernels."""
    kind, A = device_kind(geom)
    aff = np.zeros(12)
    aff[[0, 4, 8]] = 1.0
    J = None
    if kind == 2:
        aff[:9] = np.asarray(A, dtype=float).ravel()
        b = getattr(geom, "b", None)
        if b is None:  # the reference's affine_map: b = F(0)
            b = np.asarray(geom.evaluate(np.zeros((1, 3))), dtype=float)[0]
        aff[9:] = np.asarray(b, dtype=float).ravel()
    elif kind == 3:
        xi, _, _ = quad.points()
        Jh = np.asarray(geom.jacobian(xi), dtype=float).reshape(-1, 9)
        if np.any(np.linalg.det(Jh.reshape(-1, 3, 3)) <= 0):
            from .errors import DegenerateGeometryError
            raise DegenerateGeometryError(None, float("nan"), "det J <= 0 at a Gauss point")
        J, _ = _dev.to_device(Jh)
    return kind, np.ascontiguousarray(aff), J


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def assemble_rhs(space, geom, f, gauss_pts_per_span=None, out=None):
    """Load vector f_i = int det J b_i (f o F) dxi by tensor Gauss quadrature (assembly.py:201-230).

    Returns a fresh fp64 ndarray, or writes the CUDA tensor ``out`` (length n_dofs) and returns it."""
    quad = _Quad(space, gauss_pts_per_span)
    kind, aff, J = _geometry_args(geom, quad)
    case_id = getattr(f, "_mfwq_case", CASE_VALUES)
    vals = None
    if case_id == CASE_VALUES or kind == 3:
        xi, _, _ = quad.points()
        vals, _ = _dev.to_device(np.asarray(f(geom.evaluate(xi)), dtype=float).ravel())
        case_id = CASE_VALUES
    dst = out if out is not None else _dev.empty(quad.ndofs)
    if dst.numel() != quad.ndofs:
        raise ValueError(f"expected output of length {quad.ndofs}, got {dst.numel()}")
    _lib.check(_lib.lib().mfwq_quad_rhs(quad._h, kind, _lib.dptr(aff), _ptr(J), case_id, _ptr(vals),
                                        _ptr(dst), C.c_void_p(_dev.stream_ptr())))
    return dst if out is not None else dst.cpu().numpy()


def _error_integrals(space, geom, u_coeffs, case, gauss_pts, with_gradient):
    """(err2, ref2) of problems.py:97-142 on the device."""
    u, _ = _dev.to_device(u_coeffs)
    if u.numel() != space.n_dofs:
        raise ValueError(f"expected coefficient vector of length {space.n_dofs}, got {u.numel()}")
    quad = _Quad(space, gauss_pts)
    kind, aff, J = _geometry_args(geom, quad)
    case_id = getattr(case, "device_case", CASE_VALUES)
    uv = gv = None
    if case_id == CASE_VALUES or kind == 3:
        xi, _, _ = quad.points()
        x = geom.evaluate(xi)
        uv, _ = _dev.to_device(np.asarray(case.u(x), dtype=float).ravel())
        if with_gradient:
            gv, _ = _dev.to_device(np.asarray(case.grad_u(x), dtype=float).reshape(-1))
        case_id = CASE_VALUES
    er = np.zeros(2)
    _lib.check(_lib.lib().mfwq_quad_errors(quad._h, kind, _lib.dptr(aff), _ptr(J), case_id, _ptr(uv), _ptr(gv),
                                           _ptr(u), int(bool(with_gradient)), _lib.dptr(er),
                                           C.c_void_p(_dev.stream_ptr())))
    return float(er[0]), float(er[1])


def h1_relative_error(space, geom, u_coeffs, case, gauss_pts=None) -> float:
    """Relative full H1 norm of u - u_h over the physical domain (problems.py:145-150)."""
    if gauss_pts is None:
        gauss_pts = max(kv.degree for kv in space.knotvectors) + 2
    err2, ref2 = _error_integrals(space, geom, u_coeffs, case, gauss_pts, True)
    return float(np.sqrt(err2 / ref2))


def l2_relative_error(space, geom, u_coeffs, case, gauss_pts=None) -> float:
    """Relative L2 norm of u - u_h over the physical domain (problems.py:153-158)."""
    if gauss_pts is None:
        gauss_pts = max(kv.degree for kv in space.knotvectors) + 2
    err2, ref2 = _error_integrals(space, geom, u_coeffs, case, gauss_pts, False)
    return float(np.sqrt(err2 / ref2))
