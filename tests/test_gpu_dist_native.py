"""The native slab-distributed PCG (mfwq_pcg_solve_comm) on one GPU.

The in-process transport drives all P ranks of the xi3 partition from this process: the same
solver, slab kernels, halo / all-to-all messages and allreduced scalars as the NCCL transport, one
cudaMemcpyAsync per message.  1 vs P: iterations +-1 and u within the solution bar, against the
single-GPU device PCG and the reference's own runs (golden fixtures, cfg-3 vector anchors).
The NCCL transport is exercised with a one-rank group (the only multi-rank NCCL layout one GPU has).
"""
import numpy as np
import pytest
import torch

import paper_1712_08565_b200 as M
from paper_1712_08565_b200.dist import Communicator, SlabSolver

from gpu_helpers import golden_rule, relerr
from test_gpu_fullsize import ANCH, assert_matches

pytestmark = pytest.mark.gpu


def _solve(space, rule, geom, world, b, tol=1e-8):
    S = SlabSolver(space, rule, geom, Communicator.local(world))
    xs, rep = S.cg(S.owned_slices(b), tol=tol)
    return torch.cat(xs), rep


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_native_slab_pcg_matches_single_gpu(world):
    p, n_el = 3, 16
    space = M.tensor_space(p, n_el)
    rule = M.build_tensor_rule(space)
    geom = M.quarter_ring_map()
    b = torch.from_numpy(np.random.default_rng(1).standard_normal(space.n_dofs)).cuda()
    u1, r1 = M.cg(M.setup_stiffness(space, rule, geom).apply, b, M.FDPreconditioner(space).apply, tol=1e-8)
    uP, rP = _solve(space, rule, geom, world, b)
    assert rP.converged and abs(rP.iterations - r1.iterations) <= 1, (rP.iterations, r1.iterations)
    assert rP.matvecs == rP.iterations == rP.precond_applies and len(rP.residuals) == rP.iterations + 1
    assert relerr(uP.cpu().numpy(), u1.cpu().numpy()) <= 1e-11


@pytest.mark.parametrize("world", [2, 4])
def test_native_slab_pcg_thin_slabs(world):
    """Slabs thinner than p: the forward halo and the reverse halo span several owners."""
    p, n_el = 5, 8
    space = M.tensor_space(p, n_el)
    rule = M.build_tensor_rule(space)
    geom = M.quarter_ring_map()
    b = torch.from_numpy(np.random.default_rng(3).standard_normal(space.n_dofs)).cuda()
    u1, r1 = M.cg(M.setup_stiffness(space, rule, geom).apply, b, M.FDPreconditioner(space).apply, tol=1e-8)
    uP, rP = _solve(space, rule, geom, world, b)
    assert abs(rP.iterations - r1.iterations) <= 1
    assert relerr(uP.cpu().numpy(), u1.cpu().numpy()) <= 1e-10


def test_native_slab_pcg_matches_reference_golden():
    from conftest import load_golden
    g = load_golden("ring_p3_n8")
    rule, space = golden_rule(g)
    uP, rP = _solve(space, rule, M.quarter_ring_map(), 2, torch.from_numpy(g["b"]).cuda())
    assert abs(rP.iterations - int(g["iters"])) <= 1
    assert relerr(uP.cpu().numpy(), g["u"]) <= 1e-9


@pytest.mark.parametrize("world", [2, 4, 8])
def test_native_slab_pcg_cfg3(world):
    """cfg 3 (17.2 M DoFs) split over P emulated ranks against the reference's own cfg-3 run."""
    space = M.tensor_space(4, 256)
    b = torch.from_numpy(np.random.default_rng(1).standard_normal(space.n_dofs)).cuda()
    uP, rP = _solve(space, M.build_tensor_rule(space), M.quarter_ring_map(), world, b)
    a = ANCH["cfg3_u"]
    assert rP.converged and abs(rP.iterations - a["iterations"]) <= 1
    assert_matches(uP, "cfg3_u", 1e-9)


def test_native_slab_pcg_nccl_one_rank():
    """The NCCL transport over a one-rank torch.distributed group equals the device PCG."""
    import socket

    import torch.distributed as dist
    own = not dist.is_initialized()
    if own:
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        space = M.tensor_space(3, 12)
        rule = M.build_tensor_rule(space)
        geom = M.quarter_ring_map()
        b = torch.from_numpy(np.random.default_rng(1).standard_normal(space.n_dofs)).cuda()
        S = SlabSolver(space, rule, geom, Communicator.nccl())
        xs, rep = S.cg(S.owned_slices(b))
        u1, r1 = M.cg(M.setup_stiffness(space, rule, geom).apply, b, M.FDPreconditioner(space).apply)
        assert rep.iterations == r1.iterations
        assert relerr(xs[0].cpu().numpy(), u1.cpu().numpy()) <= 1e-12
    finally:
        if own:
            dist.destroy_process_group()


def test_native_slab_pcg_cfg5_one_vs_eight():
    """cfg 5 (quarter ring p = 6, n_el = 512, 137 M DoFs): the single-GPU device PCG against the same
    solve split into 8 emulated ranks (its only parity route: the CPU reference cannot run cfg 5)."""
    import gc
    space = M.tensor_space(6, 512)
    rule = M.build_tensor_rule(space)
    geom = M.quarter_ring_map()
    b = torch.from_numpy(np.random.default_rng(1).standard_normal(space.n_dofs)).cuda()
    A = M.setup_stiffness(space, rule, geom)
    P = M.FDPreconditioner(space)
    u1, r1 = M.cg(A.apply, b, P.apply, tol=1e-8)
    u1 = u1.cpu()
    del A, P
    gc.collect()
    torch.cuda.empty_cache()
    uP, rP = _solve(space, rule, geom, 8, b)
    assert r1.converged and rP.converged and abs(rP.iterations - r1.iterations) <= 1, (rP.iterations, r1.iterations)
    assert float(torch.linalg.vector_norm(uP.cpu() - u1) / torch.linalg.vector_norm(u1)) <= 1e-9
