"""Mass operator, apply_system and SystemOperator (operators.py:46-61, 87-132, 231-257;
SURVEY 8(f) rank 3) on the GPU vs the reference's own runs (tests/golden/solvers/mass_golden.npz)."""
import os

import numpy as np
import pytest
import torch

import paper_1712_08565_b200 as M
from conftest import load_golden
from gpu_helpers import geom_of, golden_rule, relerr

pytestmark = pytest.mark.gpu
Z = np.load(os.path.join(os.path.dirname(__file__), "golden", "solvers", "mass_golden.npz"))
ALPHA = {"const": 2.5, "field": lambda X: 1.0 + X[:, 0] ** 2 + 0.5 * X[:, 2]}


def _setup():
    g = load_golden("ring_p3_n8")  # uniform p=3, n_el=8: the reference's own 1D factors
    return golden_rule(g)


@pytest.mark.parametrize("gname", ["ring", "shear"])
@pytest.mark.parametrize("aname", ["const", "field"])
def test_mass_and_system_match_reference(gname, aname):
    rule, space = _setup()
    geom = geom_of(gname)
    K = M.setup_stiffness(space, rule, geom)
    Mo = M.setup_mass(space, rule, geom, alpha=ALPHA[aname])
    x = np.random.default_rng(0).standard_normal(K.n_dofs)
    meter = M.CostMeter()
    y = Mo.apply(x, meter)
    assert isinstance(y, np.ndarray)
    assert relerr(y, Z[f"{gname}_{aname}_y"]) <= 1e-12
    assert meter.flops == int(Z[f"{gname}_{aname}_flops"])
    meter = M.CostMeter()
    w = M.apply_system(Mo, K, x, meter)
    assert relerr(w, Z[f"{gname}_{aname}_sys"]) <= 1e-12
    assert meter.flops == int(Z[f"{gname}_{aname}_sysflops"])
    # device in, device out; SystemOperator is the same apply
    wd = M.SystemOperator(K, Mo).apply(torch.from_numpy(x).cuda())
    assert wd.is_cuda and relerr(wd.cpu().numpy(), w) <= 1e-14


def test_mass_on_the_fly_and_zero_alpha():
    rule, space = _setup()
    geom = geom_of("ring")
    Ms = M.setup_mass(space, rule, geom, alpha=2.5)
    Mf = M.setup_mass(space, rule, geom, alpha=2.5, on_the_fly=True)
    x = torch.from_numpy(np.random.default_rng(3).standard_normal(Ms.n_dofs)).cuda()
    assert Mf.coeff_scalars == 0 and Mf.setup_flops == 0 and Ms.coeff_scalars == Ms.n_points
    assert Mf.apply_flops == Ms.apply_flops + M.COEFF_EVAL_FLOPS * Ms.n_points
    assert relerr(Mf.apply(x).cpu().numpy(), Ms.apply(x).cpu().numpy()) <= 1e-14
    Mf.set_on_the_fly(False)
    # stored again: the same fused kernel, differing only by the order of its fp64 atomics
    assert Mf.coeff_scalars == Mf.n_points and relerr(Mf.apply(x).cpu().numpy(), Ms.apply(x).cpu().numpy()) <= 1e-14
    K = M.setup_stiffness(space, rule, geom)
    Z0 = M.setup_mass(space, rule, geom, alpha=0.0)
    m1, m2 = M.CostMeter(), M.CostMeter()
    w = M.apply_system(Z0, K, x, m1)
    # the two stiffness applies differ only by the order of fp64 atomics
    assert relerr(w.cpu().numpy(), K.apply(x, m2).cpu().numpy()) <= 1e-14 and m1.flops == m2.flops


def test_system_pcg_matches_reference():
    rule, space = _setup()
    geom = geom_of("ring")
    S = M.SystemOperator(M.setup_stiffness(space, rule, geom), M.setup_mass(space, rule, geom, alpha=2.5))
    P = M.FDPreconditioner(space, sigma=2.5)
    b = np.random.default_rng(1).standard_normal(S.n_dofs)
    u, rep = M.cg(S.apply, b, P.apply, tol=1e-8)
    it, conv, mv, pc = Z["sys_meta"].tolist()
    assert rep.converged and abs(rep.iterations - it) <= 1
    assert relerr(u, Z["sys_u"]) <= 1e-9


def test_mass_degenerate_geometry():
    rule, space = _setup()
    flip = M.GeometryMap(3, "flip", lambda xi: xi * np.array([1.0, 1.0, -1.0]),
                         lambda xi: np.broadcast_to(np.diag([1.0, 1.0, -1.0]), (len(xi), 3, 3)).copy())
    with pytest.raises(M.DegenerateGeometryError):
        M.setup_mass(space, rule, flip)


@pytest.mark.parametrize("p,n_el,gname", [(3, 8, "ring"), (5, 7, "shear"), (2, 12, "identity"), (8, 10, "ring")])
def test_fused_mass_equals_composed_path(p, n_el, gname):
    """The mass operator on the fused kernel (one term: B0 / W00 in every direction, the stored
    alpha det J grid) against the composed K1 band contractions (operators.py:87-132 step by step)."""
    from paper_1712_08565_b200 import _lib
    space = M.tensor_space(p, n_el)
    rule = M.build_tensor_rule(space)
    Mo = M.setup_mass(space, rule, geom_of(gname), alpha=ALPHA["field"])
    x = torch.from_numpy(np.random.default_rng(4).standard_normal(space.n_dofs)).cuda()
    yf = Mo.apply(x).clone()
    _lib.check(_lib.lib().mfwq_stiffness_set_path(Mo._h, 1))  # composed path
    yg = Mo.apply(x)
    assert relerr(yf.cpu().numpy(), yg.cpu().numpy()) <= 1e-13
