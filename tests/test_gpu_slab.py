"""Slab (multi-GPU) mode of the fused kernel, checked on one GPU.

Each rank's slab operator is run in turn on its input window; summing the
output windows must reproduce the whole-domain matvec (1 vs P
consistency).  No rank waits on another, so this is safe on a single device.
"""
import numpy as np
import pytest
import torch

import paper_1712_08565_b200 as M
from paper_1712_08565_b200.dist import SlabPartition, cuda_fd_dir_op

from gpu_helpers import relerr

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("p,n_el,world,kind", [(3, 16, 2, "ring"), (4, 24, 4, "ring"), (2, 12, 3, "identity"),
                                               (6, 20, 2, "ring")])
def test_slab_windows_sum_to_global(p, n_el, world, kind):
    space = M.tensor_space(p, n_el)
    rule = M.build_tensor_rule(space)
    geom = M.quarter_ring_map() if kind == "ring" else M.identity_map(3)
    A = M.setup_stiffness(space, rule, geom)
    n = A.n
    plane = n[0] * n[1]
    x = torch.from_numpy(np.random.default_rng(0).standard_normal(A.n_dofs)).cuda()
    ref = A.apply(x)
    part = SlabPartition(n_el, p, n[2], world).validate()
    y = torch.zeros_like(ref)
    for r in range(world):
        op = M.StiffnessOperator(space, rule, geom, _slab=part.elements(r))
        assert (op.slab["v_lo"], op.slab["v_hi"]) == part.in_window(r)
        assert (op.slab["y_lo"], op.slab["y_hi"]) == part.out_window(r)
        vlo, vhi = part.in_window(r)
        ylo, yhi = part.out_window(r)
        yr = op.apply(x[vlo * plane:vhi * plane])
        y[ylo * plane:yhi * plane] += yr
    assert relerr(y.cpu().numpy(), ref.cpu().numpy()) <= 1e-13


def _bent_map():
    """A general (non-analytic-kind) map whose Jacobian varies with all three coordinates: the
    operator evaluates it on the host and uploads full-domain (Nq, 3, 3) arrays (MFWQ_GEOM_JACOBIAN)."""
    def _map(xi):
        return np.stack([xi[:, 0] + 0.1 * xi[:, 1] * xi[:, 2], xi[:, 1] + 0.05 * xi[:, 0] ** 2,
                         xi[:, 2] * (1.0 + 0.2 * xi[:, 0])], axis=1)

    def _jac(xi):
        J = np.zeros((len(xi), 3, 3))
        J[:, 0, 0] = 1.0
        J[:, 0, 1] = 0.1 * xi[:, 2]
        J[:, 0, 2] = 0.1 * xi[:, 1]
        J[:, 1, 0] = 0.1 * xi[:, 0]
        J[:, 1, 1] = 1.0
        J[:, 2, 0] = 0.2 * xi[:, 2]
        J[:, 2, 2] = 1.0 + 0.2 * xi[:, 0]
        return J

    return M.GeometryMap(3, "bent", _map, _jac)


@pytest.mark.parametrize("world", [2, 3])
def test_slab_windows_sum_to_global_jacobian_and_kfield(world):
    """Slab handles read their own quadrature planes of the full-domain J and K-field arrays
    (a rank with q_lo > 0 must not reuse the bottom slab's Jacobians)."""
    p, n_el = 3, 12
    space = M.tensor_space(p, n_el)
    rule = M.build_tensor_rule(space)
    geom = _bent_map()

    def K(X):  # per-point SPD diffusion, varying along x3
        k = np.zeros((len(X), 3, 3))
        k[:, 0, 0] = 1.0 + X[:, 2] ** 2
        k[:, 1, 1] = 2.0 + X[:, 0]
        k[:, 2, 2] = 1.5 + 0.5 * np.sin(3 * X[:, 2])
        k[:, 0, 2] = k[:, 2, 0] = 0.1 * X[:, 1]
        return k

    A = M.setup_stiffness(space, rule, geom, K=K)
    n = A.n
    plane = n[0] * n[1]
    x = torch.from_numpy(np.random.default_rng(0).standard_normal(A.n_dofs)).cuda()
    ref = A.apply(x)
    part = SlabPartition(n_el, p, n[2], world).validate()
    y = torch.zeros_like(ref)
    for r in range(world):
        op = M.StiffnessOperator(space, rule, geom, K=K, _slab=part.elements(r))
        vlo, vhi = part.in_window(r)
        ylo, yhi = part.out_window(r)
        y[ylo * plane:yhi * plane] += op.apply(x[vlo * plane:vhi * plane])
    assert relerr(y.cpu().numpy(), ref.cpu().numpy()) <= 1e-13


def test_fd_dir_ops_compose_to_apply():
    space = M.tensor_space(3, 10)
    P = M.FDPreconditioner(space)
    n1, n2, n3 = P._n3
    op = cuda_fd_dir_op(P)
    x = torch.from_numpy(np.random.default_rng(2).standard_normal(P.n_dofs)).cuda()
    s = op(0, 0, 0, x, n3, n2, 0)
    s = op(1, 0, 0, s, n3, n2, 0)
    s = op(2, 0, 1, s, n3, n2, 0)
    s = op(2, 1, 0, s, n3, n2, 0)
    s = op(1, 1, 0, s, n3, n2, 0)
    s = op(0, 1, 0, s, n3, n2, 0)
    assert relerr(s.cpu().numpy(), P.apply(x).cpu().numpy()) <= 1e-13


def test_distributed_pcg_single_rank_nccl():
    """setup_distributed + dist_cg over a one-rank NCCL group on cuda:0 (the multi-GPU code path with
    its collectives degenerate) equals the single-GPU device PCG: iterations and solution."""
    import socket

    import torch.distributed as dist

    from paper_1712_08565_b200.dist import dist_cg, setup_distributed

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        p, n_el = 3, 12
        space = M.tensor_space(p, n_el)
        rule = M.build_tensor_rule(space)
        A, P, part = setup_distributed(space, rule, M.quarter_ring_map())
        assert part.owned(0) == (0, space.n_per_dir[2])
        b = torch.from_numpy(np.random.default_rng(1).standard_normal(space.n_dofs)).cuda()
        u, rep = dist_cg(A.apply, b, P.apply, tol=1e-8)
        A1 = M.setup_stiffness(space, rule, M.quarter_ring_map())
        u1, rep1 = M.cg(A1.apply, b, M.FDPreconditioner(space).apply, tol=1e-8)
        assert rep.converged and abs(rep.iterations - rep1.iterations) <= 1
        assert relerr(u.cpu().numpy(), u1.cpu().numpy()) <= 1e-9
    finally:
        dist.destroy_process_group()


def test_slab_windows_sum_to_global_deterministic():
    """Deterministic mode on slab handles (output window rows [y_lo, y_hi))."""
    p, n_el, world = 4, 16, 3
    space = M.tensor_space(p, n_el)
    rule = M.build_tensor_rule(space)
    geom = M.quarter_ring_map()
    A = M.setup_stiffness(space, rule, geom)
    A.set_deterministic(True)
    plane = A.n[0] * A.n[1]
    x = torch.from_numpy(np.random.default_rng(0).standard_normal(A.n_dofs)).cuda()
    ref = A.apply(x)
    part = SlabPartition(n_el, p, A.n[2], world).validate()
    y = torch.zeros_like(ref)
    for r in range(world):
        op = M.StiffnessOperator(space, rule, geom, _slab=part.elements(r))
        op.set_deterministic(True)
        vlo, vhi = part.in_window(r)
        ylo, yhi = part.out_window(r)
        y[ylo * plane:yhi * plane] += op.apply(x[vlo * plane:vhi * plane])
    assert relerr(y.cpu().numpy(), ref.cpu().numpy()) <= 1e-13
