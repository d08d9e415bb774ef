"""FD preconditioner and PCG on B200 (mirrors solvers.py).

``FDPreconditioner(space, sigma)`` builds the 1D exact stiffness/mass
natively (``mfwq_univariate_km``), solves the generalized eigenproblems with
cuSOLVER and applies P^-1 with fp64 tensor-core GEMMs.  ``cg`` runs the whole
loop on the device (``mfwq_pcg_solve``) when both callables are this
package's operators; otherwise it calls the given callables with device
vectors (or numpy, for numpy callables) and keeps the recurrences on the GPU.
"""

import csv
import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _dev, _lib
from .errors import EigenSolveError, IndefiniteOperatorError  # noqa: F401
from .kron import CostMeter, kron_apply


@dataclass
class KrylovReport:
    iterations: int
    residuals: list
    converged: bool
    matvecs: int
    precond_applies: int

    def write_csv(self, path):
        with open(path, "w", newline="", encoding="utf-8") as fh:
            w = csv.writer(fh)
            w.writerow(["iteration", "relative_residual"])
            for k, r in enumerate(self.residuals):
                w.writerow([k, f"{r:.16e}"])


def univariate_parametric_matrices(kv, interior=True):
    """Exact interior 1D stiffness/mass (solvers.py:48-62), built natively."""
    if not interior:
        raise NotImplementedError("only the interior (Dirichlet) matrices are built natively")
    knots = np.ascontiguousarray(kv.knots, dtype=float)
    n = len(knots) - kv.degree - 3
    K = np.empty((n, n))
    M = np.empty((n, n))
    _lib.check(_lib.lib().mfwq_univariate_km(int(kv.degree), len(knots), _lib.dptr(knots), _lib.dptr(K),
                                             _lib.dptr(M)))
    return K, M


class FDPreconditioner:
    """Exact Kronecker-sum inverse used as preconditioner (solvers.py:65-127)."""

    def __init__(self, space, sigma: float = 0.0):
        if sigma < 0:
            raise ValueError("sigma must be nonnegative")
        _dev.require_cuda()
        if space.dim != 3:
            raise NotImplementedError("the B200 FD preconditioner is three-dimensional")
        self.space = space
        self.sigma = float(sigma)
        self.K1, self.M1 = [], []
        for kv in space.knotvectors:
            K, M = univariate_parametric_matrices(kv)
            self.K1.append(np.ascontiguousarray(K))
            self.M1.append(np.ascontiguousarray(M))
        n3 = np.array([K.shape[0] for K in self.K1], dtype=np.int32)
        h = C.c_void_p()
        Kp = (_lib.dp * 3)(*[_lib.dptr(K) for K in self.K1])
        Mp = (_lib.dp * 3)(*[_lib.dptr(M) for M in self.M1])
        _lib.check(_lib.lib().mfwq_fd_create(_lib.iptr(n3), Kp, Mp, self.sigma, C.byref(h)))
        self._h = h
        self.U, self.lams = [], []
        for l in range(3):
            lam = np.empty(n3[l])
            U = np.empty((n3[l], n3[l]))
            _lib.check(_lib.lib().mfwq_fd_eigen(h, l, _lib.dptr(lam), _lib.dptr(U)))
            self.U.append(U)
            self.lams.append(lam)
        self._n3 = tuple(int(v) for v in n3)

    @property
    def n_dofs(self) -> int:
        return int(np.prod(self._n3))

    @property
    def inv_diag(self):
        """solvers.py:93-101 (host copy, computed from the eigenvalues)."""
        d = 3
        s = np.zeros(tuple(reversed(self._n3)))
        for l in range(d):
            shape = [1] * d
            shape[d - 1 - l] = self._n3[l]
            s = s + self.lams[l].reshape(shape)
        return 1.0 / (s.ravel() + self.sigma)

    def apply(self, r, meter: CostMeter | None = None, out=None):
        x, host = _dev.to_device(r, self.n_dofs)
        z = _dev.check_out(out, self.n_dofs) if out is not None else _dev.empty(self.n_dofs)
        _lib.check(_lib.lib().mfwq_fd_apply(self._h, C.c_void_p(x.data_ptr()), C.c_void_p(z.data_ptr()),
                                            C.c_void_p(_dev.stream_ptr())))
        if meter is not None:
            meter.add_flops(sum(2 * 2 * n * n * self.n_dofs // n for n in self._n3) + self.n_dofs)
        return _dev.back(z, host)

    __call__ = apply

    def apply_forward(self, v):
        """P v as a Kronecker sum (solvers.py:117-127), on the device."""
        x, host = _dev.to_device(v, self.n_dofs)
        out = _dev.zeros(self.n_dofs)
        for l in range(3):
            kron_apply([self.K1[k] if k == l else self.M1[k] for k in range(3)], x, accumulate_into=out)
        if self.sigma != 0.0:
            tmp = kron_apply(self.M1, x)
            out += self.sigma * tmp
        return _dev.back(out, host)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            _lib._lib.mfwq_fd_destroy(h)
            self._h = None


def stopping_tolerance(galerkin_rel_error: float, eta: float = 0.1) -> float:
    """solvers.py:130-134."""
    if galerkin_rel_error <= 0:
        raise ValueError("Galerkin error estimate must be positive")
    return eta * galerkin_rel_error


def _bound_op(f, cls):
    if isinstance(f, cls):
        return f
    obj = getattr(f, "__self__", None)
    if isinstance(obj, cls) and getattr(f, "__name__", "") in ("apply", "__call__"):
        return obj
    return None


def cg(apply_A, b, apply_P=None, tol=1e-8, maxit=1000, meter=None):
    """Preconditioned CG, stop on ||r||/||b|| <= tol (solvers.py:137-173)."""
    from .operators import StiffnessOperator

    A_op = _bound_op(apply_A, StiffnessOperator)
    P_op = _bound_op(apply_P, FDPreconditioner) if apply_P is not None else None
    if A_op is not None and (apply_P is None or P_op is not None):
        bt, host = _dev.to_device(b, A_op.n_dofs)
        x = _dev.empty(A_op.n_dofs)
        hist = np.zeros(maxit + 2)
        rep = _lib.KrylovReportC()
        _lib.check(_lib.lib().mfwq_pcg_solve(A_op._h, P_op._h if P_op is not None else None,
                                             C.c_void_p(bt.data_ptr()), C.c_void_p(x.data_ptr()), float(tol),
                                             int(maxit), _lib.dptr(hist), C.byref(rep),
                                             C.c_void_p(_dev.stream_ptr())))
        report = KrylovReport(rep.iterations, hist[: rep.n_residuals].tolist(), bool(rep.converged),
                              rep.matvecs, rep.precond_applies)
        return _dev.back(x, host), report
    return _cg_callables(apply_A, b, apply_P, tol, maxit)


def _cg_callables(apply_A, b, apply_P, tol, maxit):
    """Generic PCG over user callables; vectors live on the GPU."""
    import torch

    host = not _dev.is_device_tensor(b)
    bt, _ = _dev.to_device(b)

    def call(f, v):
        if host:
            return _dev.to_device(f(v.cpu().numpy()))[0]
        return _dev.to_device(f(v))[0]

    x = torch.zeros_like(bt)
    bnorm = float(torch.linalg.vector_norm(bt))
    if bnorm == 0.0:
        return _dev.back(x, host), KrylovReport(0, [0.0], True, 0, 0)
    P = apply_P if apply_P is not None else (lambda v: v)
    r = bt.clone()
    z = call(P, r)
    precs, matvecs = 1, 0
    p = z.clone()
    rz = float(r @ z)
    hist = [1.0]
    for k in range(1, maxit + 1):
        Ap = call(apply_A, p)
        matvecs += 1
        pAp = float(p @ Ap)
        if pAp <= 0:
            raise IndefiniteOperatorError(f"nonpositive curvature p.Ap = {pAp:.3e} at iteration {k}")
        alpha = rz / pAp
        x += alpha * p
        r -= alpha * Ap
        rel = float(torch.linalg.vector_norm(r)) / bnorm
        hist.append(rel)
        if rel <= tol:
            return _dev.back(x, host), KrylovReport(k, hist, True, matvecs, precs)
        z = call(P, r)
        precs += 1
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return _dev.back(x, host), KrylovReport(maxit, hist, False, matvecs, precs)


def bicgstab(apply_A, b, apply_P=None, tol=1e-8, maxit=1000, seed=0):
    """Right-preconditioned BiCGStab, true-residual history (solvers.py:176-249).

    The control flow (breakdown tests, the one seeded restart, stopping) is the
    reference's, taken on host scalars; every vector update is a fused device pass
    (``mfwq_bicg_*``, csrc/bicgstab.cu).  When ``apply_A`` / ``apply_P`` are this
    package's operators they write into persistent device buffers; other callables
    are called with device vectors (numpy callables with host copies), like ``cg``.
    The restart shadow ``r + 1e-8 |b| N(0,1)`` is drawn from numpy's
    ``default_rng(seed)`` (``seed + 1`` for the r~.v breakdown) as in the reference.
    """
    import torch

    from .operators import StiffnessOperator

    bt, host = _dev.to_device(b)
    n = bt.numel()
    L = _lib.lib()
    st = C.c_void_p(_dev.stream_ptr())

    def ptr(t):
        return C.c_void_p(t.data_ptr())

    def dot(a, c):
        out = C.c_double()
        _lib.check(L.mfwq_dot(ptr(a), ptr(c), n, C.byref(out), st))
        return out.value

    A_op = _bound_op(apply_A, StiffnessOperator)
    P_op = _bound_op(apply_P, FDPreconditioner) if apply_P is not None else None
    np_callables = host is True  # numpy in -> user callables expect numpy

    def op(f, fop, v, out):
        if fop is not None:
            return fop.apply(v, out=out)
        if np_callables:
            return _dev.to_device(f(v.cpu().numpy()), n)[0]
        return _dev.to_device(f(v), n)[0]

    def A(v, out):
        return op(apply_A, A_op, v, out)

    def P(v, out):
        if apply_P is None:
            out.copy_(v)
            return out
        return op(apply_P, P_op, v, out)

    x = torch.zeros_like(bt)
    bnorm = float(np.sqrt(dot(bt, bt)))
    if bnorm == 0.0:
        return _dev.back(x, host), KrylovReport(0, [0.0], True, 0, 0)
    eps = np.finfo(float).eps
    work = torch.empty((7, n), dtype=torch.float64, device=bt.device)
    v, p, ph, s, sh, t, tmp = work
    r = bt - A(x, tmp)
    matvecs, precs, restarted = 1, 0, False
    residuals = [1.0]
    r_shadow = r.clone()
    rho = alpha = omega = 1.0
    v.zero_()
    p.zero_()

    def restart(sd):
        noise = np.random.default_rng(sd).standard_normal(n)
        return r + (1e-8 * bnorm) * torch.from_numpy(noise).to(r.device)

    def finish(k, ok):
        return _dev.back(x, host), KrylovReport(k, residuals, ok, matvecs, precs)

    k = 0
    while k < maxit:
        k += 1
        rho_new = dot(r_shadow, r)
        if abs(rho_new) < eps * bnorm ** 2 or abs(omega) < eps:
            if restarted:
                return finish(k, False)
            restarted = True
            r_shadow = restart(seed)
            rho = alpha = omega = 1.0
            v.zero_()
            p.zero_()
            continue
        beta = (rho_new / rho) * (alpha / omega)
        rho = rho_new
        _lib.check(L.mfwq_bicg_p(ptr(p), ptr(r), ptr(v), n, beta, omega, st))
        phv = P(p, ph)
        precs += 1
        vv = A(phv, v)
        if vv.data_ptr() != v.data_ptr():
            v.copy_(vv)
        matvecs += 1
        denom = dot(r_shadow, v)
        if abs(denom) < eps * bnorm ** 2:
            if restarted:
                return finish(k, False)
            restarted = True
            r_shadow = restart(seed + 1)
            rho = alpha = omega = 1.0
            v.zero_()
            p.zero_()
            continue
        alpha = rho / denom
        ss = C.c_double()
        _lib.check(L.mfwq_bicg_s(ptr(s), ptr(r), ptr(v), n, alpha, C.byref(ss), st))
        if np.sqrt(ss.value) / bnorm <= tol:
            _lib.check(L.mfwq_axpy(ptr(x), ptr(phv), n, alpha, st))
            residuals.append(float(np.sqrt(ss.value) / bnorm))
            return finish(k, True)
        shv = P(s, sh)
        precs += 1
        tv = A(shv, t)
        matvecs += 1
        tt_ts = (C.c_double * 2)()
        _lib.check(L.mfwq_dot2(ptr(tv), ptr(s), n, tt_ts, st))
        tt, ts = tt_ts[0], tt_ts[1]
        omega = ts / tt if tt > 0 else 0.0
        rr = C.c_double()
        _lib.check(L.mfwq_bicg_xr(ptr(x), ptr(r), ptr(phv), ptr(shv), ptr(s), ptr(tv), n, alpha, omega,
                                  C.byref(rr), st))
        rel = float(np.sqrt(rr.value) / bnorm)
        residuals.append(rel)
        if rel <= tol:
            return finish(k, True)
    return finish(maxit, False)
