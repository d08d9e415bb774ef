"""Parity at the BASELINE cfg-2 size (n_el = 128, p = 2..6) against anchors produced by
running the reference itself (tests/golden/full_anchors.json, make_golden.py --full)."""
import json
import os

import numpy as np
import pytest
import torch

import paper_1712_08565_b200 as M

pytestmark = pytest.mark.gpu
ANCH = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "full_anchors.json")))
# the native WQ rule agrees with the reference lstsq to ~1e-13 (p <= 5) / ~1e-11 (p = 6)
TOL = {2: 1e-12, 3: 1e-12, 4: 1e-12, 5: 1e-12, 6: 1e-10}


@pytest.mark.parametrize("p", [2, 3, 4, 5, 6])
def test_cfg2_matvec_anchor(p):
    a = ANCH[f"cfg2_p{p}"]
    space = M.tensor_space(p, 128)
    A = M.setup_stiffness(space, M.build_tensor_rule(space), M.identity_map(3))
    assert space.n_dofs == a["N"]
    x = torch.from_numpy(np.random.default_rng(0).standard_normal(space.n_dofs)).cuda()
    y = A.apply(x).cpu().numpy()
    assert abs(np.linalg.norm(y) - a["norm_y"]) <= TOL[p] * a["norm_y"]
    head, tail = np.array(a["y_head"]), np.array(a["y_tail"])
    scale = np.abs(y).max()
    assert np.abs(y[:8] - head).max() <= TOL[p] * 1e2 * scale
    assert np.abs(y[-8:] - tail).max() <= TOL[p] * 1e2 * scale


# cfg 4 (k-method sweep, quarter ring, N = 128^3): ||u||_2 and iterations of the reference's own
# FD-PCG run on b = default_rng(1) (SURVEY §8(c) anchors, 11 significant digits)
CFG4 = {2: (128, 3.0208112873e+05, 27), 4: (126, 1.8017689318e+07, 27), 6: (124, 2.4482677025e+09, 28),
        8: (122, 4.5817363209e+11, 31), 10: (120, 1.0585471769e+14, 33)}


@pytest.mark.parametrize("p", [2, 4, 6, 8, 10])
def test_cfg4_pcg_anchor(p):
    n_el, unorm, iters = CFG4[p]
    space = M.tensor_space(p, n_el)
    A = M.setup_stiffness(space, M.build_tensor_rule(space), M.quarter_ring_map())
    P = M.FDPreconditioner(space)
    b = torch.from_numpy(np.random.default_rng(1).standard_normal(space.n_dofs)).cuda()
    u, rep = M.cg(A.apply, b, P.apply, tol=1e-8)
    assert rep.converged and abs(rep.iterations - iters) <= 1
    # anchors carry 11 digits; the solution itself is reproduced to the PCG tolerance
    assert abs(float(torch.linalg.vector_norm(u)) - unorm) <= 1e-9 * unorm


# cfg 3 (quarter ring, p = 4, n_el = 256, 17.2 M DoFs): reference anchors of SURVEY §8(c) --
# ||A x|| on x = default_rng(0), and the FD-PCG run on b = default_rng(1): 27 iterations, ||u||
CFG3_AX, CFG3_U, CFG3_IT = 1.1566850369e+01, 9.9147347659e+07, 27


@pytest.mark.parametrize("otf", [False, True])
def test_cfg3_matvec_and_pcg_anchor(otf):
    space = M.tensor_space(4, 256)
    A = M.setup_stiffness(space, M.build_tensor_rule(space), M.quarter_ring_map(), on_the_fly=otf)
    x = torch.from_numpy(np.random.default_rng(0).standard_normal(space.n_dofs)).cuda()
    ax = float(torch.linalg.vector_norm(A.apply(x)))
    assert abs(ax - CFG3_AX) <= 1e-10 * CFG3_AX  # anchor carries 11 digits
    P = M.FDPreconditioner(space)
    b = torch.from_numpy(np.random.default_rng(1).standard_normal(space.n_dofs)).cuda()
    u, rep = M.cg(A.apply, b, P.apply, tol=1e-8)
    assert rep.converged and abs(rep.iterations - CFG3_IT) <= 1
    assert abs(float(torch.linalg.vector_norm(u)) - CFG3_U) <= 1e-9 * CFG3_U
    assert rep.matvecs == rep.iterations == rep.precond_applies


def test_fd_round_trip_cfg3_size():
    """Size-independent property at the full cfg-3 size (n = 258): P^-1 (P v) = v (the reference's
    self-inverse test, test_solvers.py:35-45, at 17.2 M DoFs)."""
    space = M.tensor_space(4, 256)
    P = M.FDPreconditioner(space)
    v = torch.from_numpy(np.random.default_rng(0).standard_normal(space.n_dofs)).cuda()
    back = P.apply(P.apply_forward(v))
    assert float(torch.linalg.vector_norm(back - v)) <= 1e-10 * float(torch.linalg.vector_norm(v))
