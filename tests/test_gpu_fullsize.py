"""Parity at the BASELINE sizes against VECTOR anchors produced by running the reference itself
(tests/golden/full_vectors.json, tests/golden/make_anchors.py).

Every anchored vector (cfg 2 matvecs at p = 2..6, cfg 4 matvecs and PCG solutions at p = 2..10,
cfg 3 matvec / FD apply / PCG solution) is pinned by its 2-norm, the norm of each of its n3 xi3
planes and its dot products with 8 seeded N(0,1) probe vectors, each compared relative to ||v||.
All operators here are built by the package's own setup path (build_tensor_rule -> setup_stiffness,
FDPreconditioner), the drop-in path of operators.py:185-204 / solvers.py:107-115 / :137-173.
Bars (north_star): matvec 1e-12, solution 1e-9, PCG iterations +-1.
"""
import json
import os

import numpy as np
import pytest
import torch

import paper_1712_08565_b200 as M

pytestmark = pytest.mark.gpu
ANCH = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "full_vectors.json")))
PROBE_SEED0 = 100  # make_anchors.py
MATVEC_TOL, U_TOL = 1e-12, 1e-9


def assert_matches(v, key, tol):
    """Fingerprint comparison of a device vector against a reference anchor (make_anchors.py)."""
    a = ANCH[key]
    v = v.reshape(-1)
    assert v.numel() == a["N"]
    ref = a["norm"]
    nrm = float(torch.linalg.vector_norm(v))
    assert abs(nrm - ref) <= tol * ref, (key, "norm", abs(nrm - ref) / ref)
    n3 = len(a["planes"])
    planes = torch.linalg.vector_norm(v.reshape(n3, -1), dim=1).cpu().numpy()
    dp = np.abs(planes - np.array(a["planes"])).max() / ref
    assert dp <= tol, (key, "planes", dp)
    for k, (d, rn) in enumerate(zip(a["dots"], a["probe_norms"])):
        r = torch.from_numpy(np.random.default_rng(PROBE_SEED0 + k).standard_normal(a["N"])).to(v.device)
        got = float(torch.dot(r, v))
        assert abs(got - d) <= tol * ref * rn, (key, "dot", k, abs(got - d) / (ref * rn))


def _x(n):
    return torch.from_numpy(np.random.default_rng(0).standard_normal(n)).cuda()


def _b(n):
    return torch.from_numpy(np.random.default_rng(1).standard_normal(n)).cuda()


@pytest.mark.parametrize("p", [2, 3, 4, 5, 6])
def test_cfg2_matvec_vector_anchor(p):
    space = M.tensor_space(p, 128)
    A = M.setup_stiffness(space, M.build_tensor_rule(space), M.identity_map(3))
    assert_matches(A.apply(_x(space.n_dofs)), f"cfg2_p{p}_Ax", MATVEC_TOL)
    if p == 4:
        P = M.FDPreconditioner(space)
        assert_matches(P.apply(_x(space.n_dofs)), "cfg2_p4_fd", 1e-11)


CFG4 = {2: 128, 4: 126, 6: 124, 8: 122, 10: 120}


@pytest.mark.parametrize("p", [2, 4, 6, 8, 10])
def test_cfg4_matvec_and_pcg_vector_anchor(p):
    """k-method sweep (quarter ring, N = 128^3): the product rule at every degree incl. 8 and 10."""
    space = M.tensor_space(p, CFG4[p])
    A = M.setup_stiffness(space, M.build_tensor_rule(space), M.quarter_ring_map())
    assert_matches(A.apply(_x(space.n_dofs)), f"cfg4_p{p}_Ax", MATVEC_TOL)
    P = M.FDPreconditioner(space)
    u, rep = M.cg(A.apply, _b(space.n_dofs), P.apply, tol=1e-8)
    a = ANCH[f"cfg4_p{p}_u"]
    assert rep.converged and abs(rep.iterations - a["iterations"]) <= 1, (rep.iterations, a["iterations"])
    assert_matches(u, f"cfg4_p{p}_u", U_TOL)


@pytest.mark.parametrize("otf", [False, True])
def test_cfg3_matvec_fd_and_pcg_vector_anchor(otf):
    """cfg 3 (quarter ring, p = 4, n_el = 256, 17.2 M DoFs), stored grids and on the fly."""
    space = M.tensor_space(4, 256)
    A = M.setup_stiffness(space, M.build_tensor_rule(space), M.quarter_ring_map(), on_the_fly=otf)
    assert_matches(A.apply(_x(space.n_dofs)), "cfg3_Ax", MATVEC_TOL)
    P = M.FDPreconditioner(space)
    if not otf:
        assert_matches(P.apply(_x(space.n_dofs)), "cfg3_fd", 1e-11)
    u, rep = M.cg(A.apply, _b(space.n_dofs), P.apply, tol=1e-8)
    a = ANCH["cfg3_u"]
    assert rep.converged and abs(rep.iterations - a["iterations"]) <= 1
    assert rep.matvecs == rep.iterations == rep.precond_applies
    assert_matches(u, "cfg3_u", U_TOL)


def test_cfg3_pcg_deterministic_iterations():
    """The fused matvec accumulates w with fp64 atomics (order-dependent rounding): ten cfg-3 solves
    must still take the same number of iterations and agree to far below the solution bar."""
    space = M.tensor_space(4, 256)
    A = M.setup_stiffness(space, M.build_tensor_rule(space), M.quarter_ring_map())
    P = M.FDPreconditioner(space)
    b = _b(space.n_dofs)
    its, us = [], []
    for _ in range(10):
        u, rep = M.cg(A.apply, b, P.apply, tol=1e-8)
        its.append(rep.iterations)
        us.append(u)
    assert len(set(its)) == 1, its
    ref = us[0]
    worst = max(float(torch.linalg.vector_norm(u - ref) / torch.linalg.vector_norm(ref)) for u in us[1:])
    assert worst <= 1e-12, worst
    # deterministic accumulation (set_deterministic): the solves agree bit for bit
    A.set_deterministic(True)
    u1, r1 = M.cg(A.apply, b, P.apply, tol=1e-8)
    u2, r2 = M.cg(A.apply, b, P.apply, tol=1e-8)
    assert r1.iterations == r2.iterations == its[0] and torch.equal(u1, u2) and r1.residuals == r2.residuals
    assert_matches(u1, "cfg3_u", U_TOL)


def test_fd_round_trip_cfg3_size():
    """Size-independent property at the full cfg-3 size (n = 258): P^-1 (P v) = v (the reference's
    self-inverse test, test_solvers.py:35-45, at 17.2 M DoFs)."""
    space = M.tensor_space(4, 256)
    P = M.FDPreconditioner(space)
    v = _x(space.n_dofs)
    back = P.apply(P.apply_forward(v))
    assert float(torch.linalg.vector_norm(back - v)) <= 1e-10 * float(torch.linalg.vector_norm(v))
