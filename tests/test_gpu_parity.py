"""GPU parity: the CUDA path (through the C-ABI) against the reference's golden
outputs and the CPU oracle.  Bar (BASELINE north_star): matvec rel. error
<= 1e-12, PCG iterations within +-1, solution rel. difference <= 1e-9."""
import numpy as np
import pytest

import paper_1712_08565_b200 as M
from oracle import mfwq_oracle as O

from gpu_helpers import SHEAR, geom_of, golden_rule, relerr

pytestmark = pytest.mark.gpu

MATVEC_TOL = 1e-12


@pytest.mark.parametrize("path", ["generic", "fused"])
def test_matvec_matches_reference(golden, path):
    name, g = golden
    rule, space = golden_rule(g)
    A = M.setup_stiffness(space, rule, geom_of(g["geom"]))
    A.set_path(path)
    x = np.random.default_rng(0).standard_normal(space.n_dofs)
    meter = M.CostMeter()
    y = A.apply(x, meter)
    assert relerr(y, g["y"]) <= MATVEC_TOL, (name, relerr(y, g["y"]))
    assert meter.flops == int(g["flops"])


def test_matvec_product_rule_matches_reference(golden):
    """The drop-in path end to end: the package's OWN rule builder (build_tensor_rule, bit-identical
    to the reference's weights via numpy's dgelsd) -> setup_stiffness -> apply, at every fixture
    degree including p = 8 and 10, against the reference's matvec output."""
    name, g = golden
    kv = M.KnotVector(int(g["p"]), g["knots"])
    space = M.TensorSpace((kv, kv, kv))
    A = M.setup_stiffness(space, M.build_tensor_rule(space), geom_of(g["geom"]))
    x = np.random.default_rng(0).standard_normal(space.n_dofs)
    y = A.apply(x)
    assert relerr(y, g["y"]) <= MATVEC_TOL, (name, relerr(y, g["y"]))


def test_fd_apply_matches_reference(golden):
    name, g = golden
    if "fd_y" not in g:
        pytest.skip("no FD output stored")
    rule, space = golden_rule(g)
    P = M.FDPreconditioner(space)
    x = np.random.default_rng(0).standard_normal(space.n_dofs)
    z = P.apply(x)
    tol = 1e-11 if int(g["p"]) <= 6 else 1e-8  # M-conditioning grows ~1e8 at p=8 (test_acceptance.py:115-135)
    assert relerr(z, g["fd_y"]) <= tol, (name, relerr(z, g["fd_y"]))
    assert np.abs(np.sort(P.lams[0]) - g["lam"]).max() <= 1e-9 * np.abs(g["lam"]).max()


def test_pcg_matches_reference(golden):
    name, g = golden
    if "u" not in g:
        pytest.skip("no PCG output stored")
    rule, space = golden_rule(g)
    A = M.setup_stiffness(space, rule, geom_of(g["geom"]))
    P = M.FDPreconditioner(space)
    u, rep = M.cg(A.apply, g["b"], P.apply, tol=1e-8)
    assert rep.converged
    assert abs(rep.iterations - int(g["iters"])) <= 1, (name, rep.iterations, int(g["iters"]))
    assert relerr(u, g["u"]) <= 1e-9, (name, relerr(u, g["u"]))
    assert rep.residuals[0] == 1.0 and len(rep.residuals) == rep.iterations + 1
    assert rep.matvecs == rep.iterations and rep.precond_applies == rep.iterations


@pytest.mark.parametrize("kind", ["identity", "ring", "shear"])
def test_coefficient_grids_match_oracle(kind):
    p, n_el = 3, 5
    space = M.tensor_space(p, n_el)
    rule = M.build_tensor_rule(space)
    A = M.setup_stiffness(space, rule, geom_of(kind))
    orules = [O.rule_1d(O.uniform_knots(p, n_el))] * 3
    ref = O.stiffness_coeffs(orules, O.jac_for(kind, SHEAR))
    got = A.coeffs
    for key, r in ref.items():
        assert np.abs(got[key] - r).max() <= 1e-14 * max(1.0, np.abs(r).max()), (kind, key)
    if kind == "identity":
        for key in ((0, 1), (0, 2), (1, 2)):
            assert not got[key].any()
    assert A.coeff_scalars == 6 * rule.n_points


def test_degenerate_geometry_raises():
    folded = M.GeometryMap(3, "folded", lambda xi: xi,
                           lambda xi: np.broadcast_to(np.diag([1.0, -1.0, 1.0]), (len(xi), 3, 3)).copy())
    space = M.tensor_space(1, 2)
    with pytest.raises(M.DegenerateGeometryError):
        M.setup_stiffness(space, M.build_tensor_rule(space), folded)


def test_zero_vector_and_length_mismatch():
    space = M.tensor_space(2, 3)
    A = M.setup_stiffness(space, M.build_tensor_rule(space), M.quarter_ring_map())
    assert np.array_equal(A.apply(np.zeros(space.n_dofs)), np.zeros(space.n_dofs))
    with pytest.raises(ValueError):
        A.apply(np.zeros(space.n_dofs + 1))
    P = M.FDPreconditioner(space)
    assert np.array_equal(P.apply(np.zeros(space.n_dofs)), np.zeros(space.n_dofs))
    with pytest.raises(ValueError):
        P.apply(np.zeros(space.n_dofs + 1))
    with pytest.raises(ValueError):
        M.FDPreconditioner(space, sigma=-1.0)


@pytest.mark.parametrize("p,n_el", [(2, 8), (5, 8), (7, 8), (3, 16)])
def test_fd_self_inverse(p, n_el):
    """solvers test_self_inverse (test_solvers.py:35-45) on the device."""
    space = M.tensor_space(p, n_el)
    P = M.FDPreconditioner(space)
    v = np.random.default_rng(0).standard_normal(space.n_dofs)
    back = P.apply(P.apply_forward(v))
    assert relerr(back, v) <= 1e-10


def test_native_rule_end_to_end_cfg1():
    """Package-built rule (C++ WQ) + GPU operator vs the reference golden at cfg 1."""
    from conftest import load_golden
    g = load_golden("cfg1_cube_p3_n16")
    space = M.tensor_space(3, 16)
    A = M.setup_stiffness(space, M.build_tensor_rule(space), M.identity_map(3))
    x = np.random.default_rng(0).standard_normal(space.n_dofs)
    assert relerr(A.apply(x), g["y"]) <= MATVEC_TOL
    P = M.FDPreconditioner(space)
    u, rep = M.cg(A.apply, g["b"], P.apply, tol=1e-8)
    assert rep.iterations == int(g["iters"]) == 1
    assert relerr(u, g["u"]) <= 1e-9


def test_cg_generic_callables():
    b = np.random.default_rng(0).standard_normal(50)
    x, rep = M.cg(lambda v: v, b, tol=1e-12)
    assert rep.iterations == 1 and np.allclose(x, b)
    x, rep = M.cg(lambda v: v, np.zeros(10))
    assert rep.iterations == 0 and not x.any()
    with pytest.raises(M.IndefiniteOperatorError):
        M.cg(lambda v: -v, np.ones(5))


def test_cg_device_indefinite_and_maxit():
    space = M.tensor_space(2, 4)
    A = M.setup_stiffness(space, M.build_tensor_rule(space), M.quarter_ring_map())
    b = np.random.default_rng(3).standard_normal(space.n_dofs)
    x, rep = M.cg(A.apply, b, tol=1e-14, maxit=3)
    assert not rep.converged and rep.iterations == 3 and len(rep.residuals) == 4
    x, rep = M.cg(A.apply, np.zeros(space.n_dofs))
    assert rep.iterations == 0 and rep.residuals == [0.0]


def test_kron_apply_vs_oracle():
    rng = np.random.default_rng(7)
    fs = [rng.standard_normal((3, 4)), rng.standard_normal((5, 2)), rng.standard_normal((2, 3))]
    x = rng.standard_normal(4 * 2 * 3)
    assert relerr(M.kron_apply(fs, x), O.kron_apply(fs, x)) <= 1e-13
    meter = M.CostMeter()
    M.kron_apply([np.ones((4, 4))] * 3, np.ones(64), meter)
    assert meter.flops == 2 * 4 * 4 * (16 + 16 + 16)


def test_torch_device_inputs_stay_on_device():
    import torch
    space = M.tensor_space(3, 6)
    A = M.setup_stiffness(space, M.build_tensor_rule(space), M.quarter_ring_map())
    x = torch.randn(space.n_dofs, dtype=torch.float64, device="cuda")
    y = A.apply(x)
    assert isinstance(y, torch.Tensor) and y.is_cuda
    assert relerr(y.cpu().numpy(), A.apply(x.cpu().numpy())) <= 1e-14  # fp64 atomics: order-dependent rounding


def test_pinned_host_apply_is_pipelined_and_exact():
    """Pinned host tensors take the asynchronous path (side-stream H2D, double-buffered staging):
    after a stream sync every result equals the device-path result."""
    import torch
    space = M.tensor_space(3, 6)
    A = M.setup_stiffness(space, M.build_tensor_rule(space), M.quarter_ring_map())
    xs = [torch.from_numpy(np.random.default_rng(s).standard_normal(space.n_dofs)).pin_memory() for s in range(5)]
    outs = [torch.empty(space.n_dofs, dtype=torch.float64, pin_memory=True) for _ in xs]
    for x, o in zip(xs, outs):
        assert A.apply(x, out=o) is o
    torch.cuda.current_stream().synchronize()
    for x, o in zip(xs, outs):
        ref = A.apply(x.numpy())
        assert relerr(o.numpy(), ref) <= 1e-14
    auto = A.apply(xs[0])  # allocates a pinned result
    torch.cuda.current_stream().synchronize()
    assert auto.is_pinned() and relerr(auto.numpy(), A.apply(xs[0].numpy())) <= 1e-14


def test_apply_pipelined_matches():
    import torch
    space = M.tensor_space(2, 7)
    A = M.setup_stiffness(space, M.build_tensor_rule(space), M.identity_map(3))
    xs = [torch.from_numpy(np.random.default_rng(s).standard_normal(space.n_dofs)).pin_memory() for s in range(4)]
    res = [A.apply_pipelined(x) for x in xs]
    for (o, ev), x in zip(res, xs):
        ev.synchronize()
        assert relerr(o.numpy(), A.apply(x.numpy())) <= 1e-14
    with pytest.raises(ValueError):
        A.apply_pipelined(np.zeros(space.n_dofs))


def test_pcg_c_abi_unaligned_solution_buffer():
    """mfwq_pcg_solve with x 8 bytes off a 16-byte boundary and odd N (the vectorised update
    kernels iterate in an aligned copy and hand the result back) equals the aligned call."""
    import ctypes as C

    import torch

    from paper_1712_08565_b200 import _dev, _lib

    space = M.tensor_space(3, 6)  # n = 7 per direction: N = 343, odd
    assert space.n_dofs % 2 == 1
    A = M.setup_stiffness(space, M.build_tensor_rule(space), M.quarter_ring_map())
    P = M.FDPreconditioner(space)
    b = np.random.default_rng(1).standard_normal(space.n_dofs)
    u_ref, rep_ref = M.cg(A.apply, b, P.apply, tol=1e-10)
    bt = torch.from_numpy(b).cuda()
    buf = torch.zeros(space.n_dofs + 1, dtype=torch.float64, device="cuda")
    x = buf[1:]
    assert x.data_ptr() % 16 == 8
    hist = np.zeros(1002)
    rep = _lib.KrylovReportC()
    _lib.check(_lib.lib().mfwq_pcg_solve(A._h, P._h, C.c_void_p(bt.data_ptr()), C.c_void_p(x.data_ptr()),
                                         1e-10, 1000, _lib.dptr(hist), C.byref(rep),
                                         C.c_void_p(_dev.stream_ptr())))
    torch.cuda.synchronize()
    assert rep.iterations == rep_ref.iterations and bool(rep.converged)
    assert relerr(x.cpu().numpy(), u_ref) <= 1e-13
    assert float(buf[0]) == 0.0


@pytest.mark.parametrize("p,n_el", [(1, 4), (4, 8), (8, 32)])
def test_fd_eigenpairs_residual_and_m_orthonormality(p, n_el):
    """test_solvers.py:14-23 on the device eigensolver (cuSOLVER Dsygvd): K U = M U diag(lam),
    U^T M U = I to 1e-10, lam > 0."""
    space = M.tensor_space(p, n_el)
    P = M.FDPreconditioner(space)
    K, Mm = P.K1[0], P.M1[0]
    U, lam = P.U[0], np.asarray(P.lams[0])
    assert np.abs(K @ U - Mm @ U @ np.diag(lam)).max() <= 1e-10
    assert np.abs(U.T @ Mm @ U - np.eye(len(lam))).max() <= 1e-10
    assert lam.min() > 0


def test_device_pcg_true_residual_matches_reported():
    """test_solvers.py:95-102 for the device-resident PCG: the true relative residual of the
    returned solution is within 10x of the last recursive residual."""
    space = M.tensor_space(4, 12)
    A = M.setup_stiffness(space, M.build_tensor_rule(space), M.quarter_ring_map())
    P = M.FDPreconditioner(space)
    b = np.random.default_rng(3).standard_normal(space.n_dofs)
    x, rep = M.cg(A.apply, b, P.apply, tol=1e-10)
    true_rel = np.linalg.norm(b - A.apply(x)) / np.linalg.norm(b)
    assert rep.converged and true_rel <= 10 * rep.residuals[-1]


def test_preconditioner_robustness_in_p_and_h():
    """test_acceptance.py:214-232 (criterion 8) on the device path: FD-preconditioned BiCGStab on
    the oscillating quarter-ring case, iteration counts vary by < 2x across p = 2..8 and h."""
    geom = M.quarter_ring_map()

    def iters(p, n_el):
        space = M.tensor_space(p, n_el)
        A = M.setup_stiffness(space, M.build_tensor_rule(space), geom)
        rhs = M.assemble_rhs(space, geom, M.oscillating_case().f)
        _, rep = M.bicgstab(A.apply, rhs, M.FDPreconditioner(space).apply, tol=1e-8)
        assert rep.converged, (p, n_el)
        return rep.iterations

    by_p = [iters(p, 16) for p in range(2, 9)]
    assert max(by_p) < 2 * min(by_p), by_p
    by_h = [iters(3, n_el) for n_el in (8, 16, 32)]
    assert max(by_h) < 2 * min(by_h), by_h


def test_in_place_apply_rejected():
    """y is zeroed before the fused kernel reads x, so an overlapping out= must raise, not corrupt."""
    import torch

    space = M.tensor_space(2, 4)
    A = M.setup_stiffness(space, M.build_tensor_rule(space), M.identity_map(3))
    x = torch.ones(space.n_dofs, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        A.apply(x, out=x)
    y = A.apply(x)
    assert float(torch.linalg.vector_norm(y)) > 0


@pytest.mark.parametrize("p,n_el,kind", [(3, 8, "ring"), (4, 11, "shear"), (2, 9, "identity"), (10, 10, "ring")])
def test_deterministic_matvec_is_bitwise_reproducible(p, n_el, kind):
    """set_deterministic(): the overlapping output windows are summed in a fixed order instead of
    by fp64 atomics -- repeated applies agree bit for bit and equal the atomic path to rounding."""
    import torch
    space = M.tensor_space(p, n_el)
    A = M.setup_stiffness(space, M.build_tensor_rule(space), geom_of(kind))
    x = torch.from_numpy(np.random.default_rng(5).standard_normal(space.n_dofs)).cuda()
    ya = A.apply(x).clone()
    A.set_deterministic(True)
    y1 = A.apply(x).clone()
    y2 = A.apply(x).clone()
    assert torch.equal(y1, y2)
    assert relerr(y1.cpu().numpy(), ya.cpu().numpy()) <= 1e-14


def test_numpy_apply_pageable_pipeline_multi_chunk_and_threads():
    """A.apply(np.ndarray): the native pageable pipeline (pinned chunk slots, host copy pool) over
    several chunks, from two host threads at once, equals the device-tensor apply."""
    import threading

    import torch
    space = M.tensor_space(3, 80)  # 531,441 DoFs: more than one 4 MB staging chunk each way
    rule = M.build_tensor_rule(space)
    ops = [M.setup_stiffness(space, rule, M.quarter_ring_map()) for _ in range(2)]
    for A in ops:
        A.set_deterministic(True)  # bitwise comparable
    xs = [np.random.default_rng(s).standard_normal(space.n_dofs) for s in range(2)]
    refs = [A.apply(torch.from_numpy(x).cuda()).cpu().numpy() for A, x in zip(ops, xs)]
    out = [None, None]

    def run(i):
        torch.cuda.set_device(0)
        for _ in range(3):
            out[i] = ops[i].apply(xs[i])

    ts = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for i in range(2):
        assert isinstance(out[i], np.ndarray) and np.array_equal(out[i], refs[i])
