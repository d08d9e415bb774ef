"""BiCGStab (solvers.py:176-249) on the GPU vs the reference's own runs
(tests/golden/solvers/bicgstab_golden.npz, made by tests/golden/make_golden.py):
FD-preconditioned convergence, the maxit report, and the breakdown -> seeded restart ->
failure path on a skew operator, through numpy and device callables."""
import os

import numpy as np
import pytest
import torch

import paper_1712_08565_b200 as M
from conftest import load_golden
from gpu_helpers import geom_of, golden_rule, relerr

pytestmark = pytest.mark.gpu
Z = np.load(os.path.join(os.path.dirname(__file__), "golden", "solvers", "bicgstab_golden.npz"))


def _check(tag, x, rep, iter_slack=0, xtol=1e-9):
    it, conv, mv, pc = Z[f"{tag}_meta"].tolist()
    assert rep.converged == bool(conv), tag
    assert abs(rep.iterations - it) <= iter_slack, (tag, rep.iterations, it)
    if iter_slack == 0:
        assert (rep.matvecs, rep.precond_applies) == (mv, pc), tag
        assert len(rep.residuals) == len(Z[f"{tag}_hist"])
        assert np.allclose(rep.residuals, Z[f"{tag}_hist"], rtol=1e-6, atol=1e-12), tag
    xr = Z[f"{tag}_x"]
    xx = x.cpu().numpy() if isinstance(x, torch.Tensor) else x
    assert relerr(xx, xr) <= xtol, (tag, relerr(xx, xr))


def _ring():
    g = load_golden("ring_p3_n8")
    rule, space = golden_rule(g)
    A = M.setup_stiffness(space, rule, geom_of("ring"))
    return A, M.FDPreconditioner(space), np.random.default_rng(1).standard_normal(A.n_dofs)


def test_bicgstab_fd_matches_reference():
    A, P, b = _ring()
    x, rep = M.bicgstab(A.apply, b, P.apply, tol=1e-8)
    _check("ring_fd", x, rep, iter_slack=1)
    assert rep.residuals[0] == 1.0 and rep.residuals[-1] <= 1e-8
    # device in, device out
    xd, repd = M.bicgstab(A.apply, torch.from_numpy(b).cuda(), P.apply, tol=1e-8)
    assert xd.is_cuda and repd.iterations == rep.iterations
    assert relerr(xd.cpu().numpy(), x) <= 1e-12


def test_bicgstab_maxit_report():
    A, _, b = _ring()
    x, rep = M.bicgstab(A.apply, b, None, tol=1e-8, maxit=5)
    _check("ring_nop_maxit5", x, rep)


def _skew_np(v):
    y = np.empty_like(v)
    y[0::2] = -v[1::2]
    y[1::2] = v[0::2]
    return y


def _skew_dev(v):
    y = torch.empty_like(v)
    y[0::2] = -v[1::2]
    y[1::2] = v[0::2]
    return y


def test_bicgstab_breakdown_restart_then_failure():
    b = Z["skew_b"]
    # the iterate has diverged (residual ~3e8) when the second breakdown stops it, so rounding
    # differences are amplified: counters and history are exact, x agrees to 1e-6
    x, rep = M.bicgstab(_skew_np, b, tol=1e-8)
    _check("skew", x, rep, xtol=1e-6)
    xd, repd = M.bicgstab(_skew_dev, torch.from_numpy(b).cuda(), tol=1e-8)
    _check("skew", xd, repd, xtol=1e-6)


def test_bicgstab_zero_rhs():
    A, P, b = _ring()
    x, rep = M.bicgstab(A.apply, np.zeros_like(b), P.apply)
    assert not np.any(x) and (rep.iterations, rep.residuals, rep.converged, rep.matvecs,
                              rep.precond_applies) == (0, [0.0], True, 0, 0)
