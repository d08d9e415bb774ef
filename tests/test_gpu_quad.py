"""GPU parity of the load vector and the L2 / H1 error norms (csrc/quadrature.cu through the C-ABI)
against the reference's own outputs (tests/golden/quad).  Integrands: the built-in device cases, host
callables (values at the mapped Gauss points) and a Jacobian-only geometry."""
from types import SimpleNamespace

import numpy as np
import pytest

import paper_1712_08565_b200 as M
from oracle import mfwq_oracle as O
from quad_helpers import SHEAR, load_quad, quad_names

pytestmark = pytest.mark.gpu


def _setup(g):
    kv = M.KnotVector(g["p"], g["knots"])
    space = M.TensorSpace((kv, kv, kv))
    geom = {"identity": M.identity_map(3), "ring": M.quarter_ring_map(),
            "shear": M.affine_map(np.array(SHEAR), g["shear_b"])}[g["geom"]]
    case = M.cube_sine_case() if g["case"] == "cube" else M.oscillating_case()
    return space, geom, case


def _jacobian_only(geom):
    """The same map seen as an arbitrary geometry: Jacobians and points come from the host."""
    return SimpleNamespace(kind="custom", evaluate=geom.evaluate, jacobian=geom.jacobian)


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - b) / np.linalg.norm(b)


@pytest.mark.parametrize("name", quad_names())
@pytest.mark.parametrize("mode", ["device-case", "host-values", "jacobian-geometry"])
def test_rhs_matches_reference(name, mode):
    g = load_quad(name)
    space, geom, case = _setup(g)
    f = case.f
    if mode == "host-values":
        f = lambda x: case.f(x)  # an untagged callable: evaluated on the host at the mapped points
    if mode == "jacobian-geometry":
        geom = _jacobian_only(geom)
    rhs = M.assemble_rhs(space, geom, f, gauss_pts_per_span=None if g["rhs_gpts"] < 0 else g["rhs_gpts"])
    assert rhs.shape == (space.n_dofs,) and rhs.dtype == np.float64
    assert _rel(rhs, g["rhs"]) <= 1e-12, (name, mode, _rel(rhs, g["rhs"]))


@pytest.mark.parametrize("name", quad_names())
@pytest.mark.parametrize("mode", ["device-case", "host-values", "jacobian-geometry"])
def test_error_norms_match_reference(name, mode):
    g = load_quad(name)
    space, geom, case = _setup(g)
    if mode == "host-values":
        case = SimpleNamespace(u=case.u, grad_u=case.grad_u)  # e.g. the reference's ManufacturedCase
    if mode == "jacobian-geometry":
        geom = _jacobian_only(geom)
    from paper_1712_08565_b200.problems import _error_integrals
    for with_grad, key in ((False, "err_l2"), (True, "err_h1")):
        e2, r2 = _error_integrals(space, geom, g["u"], case, g["p"] + 2, with_grad)
        ref = g[key]
        assert abs(e2 - ref[0]) <= 1e-11 * ref[0] and abs(r2 - ref[1]) <= 1e-11 * ref[1], (name, mode, key)
    assert abs(M.l2_relative_error(space, geom, g["u"], case) - float(g["l2"])) <= 1e-11 * float(g["l2"])
    assert abs(M.h1_relative_error(space, geom, g["u"], case) - float(g["h1"])) <= 1e-11 * float(g["h1"])


def test_rhs_into_device_tensor_and_errors_on_device_vector():
    import torch
    g = load_quad("cube_p3_n4")
    space, geom, case = _setup(g)
    out = torch.empty(space.n_dofs, dtype=torch.float64, device="cuda")
    r = M.assemble_rhs(space, geom, case.f, out=out)
    assert r is out and _rel(out.cpu().numpy(), g["rhs"]) <= 1e-12
    u = torch.from_numpy(g["u"]).cuda()
    assert abs(M.h1_relative_error(space, geom, u, case) - float(g["h1"])) <= 1e-11 * float(g["h1"])


def test_cfg1_convergence_study_on_device():
    """BASELINE cfg 1 end to end on the GPU: device RHS -> FD-PCG -> device H1 error, against the oracle."""
    p, n_el = 3, 16
    space = M.tensor_space(p, n_el)
    geom = M.identity_map(3)
    case = M.cube_sine_case()
    rhs = M.assemble_rhs(space, geom, case.f)
    A = M.setup_stiffness(space, M.build_tensor_rule(space), geom)
    u, rep = M.cg(A.apply, rhs, M.FDPreconditioner(space).apply, tol=1e-8)
    assert rep.converged and rep.iterations <= 3
    kv = O.uniform_knots(p, n_el)
    ou, og, of = O.cube_sine()
    rhs_o = O.assemble_rhs([kv] * 3, lambda xi: xi.copy(), O.jac_identity, of)
    assert _rel(rhs, rhs_o) <= 1e-12
    e2, r2 = O.error_integrals([kv] * 3, lambda xi: xi.copy(), O.jac_identity, u, ou, og, p + 2, True)
    h1 = M.h1_relative_error(space, geom, u, case)
    assert abs(h1 - np.sqrt(e2 / r2)) <= 1e-10 * h1
    assert h1 < 1e-3  # p = 3 on 16^3 elements resolves the sine


def test_input_validation():
    g = load_quad("cube_p3_n4")
    space, geom, case = _setup(g)
    with pytest.raises(ValueError):
        M.l2_relative_error(space, geom, np.zeros(space.n_dofs + 1), case)
