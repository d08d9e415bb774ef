"""Multi-process (gloo, CPU) tests of the slab decomposition (paper_1712_08565_b200.dist).

The exchange protocol, window arithmetic and the distributed FD/PCG are the
same code that runs over NCCL on GPUs; here the local compute is the CPU oracle
restricted to a rank's z-elements, and the assembled results are compared with
the oracle's global matvec / FD apply / PCG (1 vs P consistency).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import mfwq_oracle as O
from paper_1712_08565_b200.dist import DistFD, DistStiffness, SlabPartition, dist_cg


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(p, n_el, kind="ring"):
    kv = O.uniform_knots(p, n_el)
    rule = O.rule_1d(kv)
    rules = [rule] * 3
    C = O.stiffness_coeffs(rules, O.jac_for(kind, np.eye(3)))
    return kv, rules, C, O.Stiffness(rules, C)


def oracle_slab_apply(rules, C, part, rank):
    """CPU stand-in for the slab kernel: only the rank's quadrature planes contribute."""
    kv = rules[2].kv
    n = [r.kv.nfun - 2 for r in rules]
    plane = n[0] * n[1]
    e0, e1 = part.elements(rank)
    # element of each quadrature point (right-continuous, last point in the last element)
    el = np.array([min(kv.span(x) - kv.p, n_el_of(kv) - 1) for x in rules[2].pts])
    q_in_slab = (el >= e0) & (el < e1)
    op = O.Stiffness(rules, C)
    for b in range(3):
        Bz = op.Bf[b][2].tolil()
        Bz[np.flatnonzero(~q_in_slab), :] = 0.0
        op.Bf[b][2] = Bz.tocsr()
    vlo, vhi = part.in_window(rank)
    ylo, yhi = part.out_window(rank)
    N = op.N

    def apply(xin):
        x = np.zeros(N)
        x[vlo * plane:vhi * plane] = xin.numpy()
        y = op.apply(x)
        outside = np.concatenate([y[:ylo * plane], y[yhi * plane:]])
        assert np.abs(outside).max(initial=0.0) == 0.0, "slab wrote outside its predicted window"
        return torch.from_numpy(y[ylo * plane:yhi * plane].copy())
    return apply


def n_el_of(kv):
    return len(kv.brk) - 1


def oracle_dir_op(fd):
    lam, U = fd.lam, fd.U

    def op(d, inverse, scale, x, nz, ny, row_lo):
        X = x.numpy().reshape(nz, ny, -1)
        A = U[d] if inverse else U[d].T  # forward: y_k = sum_i U[i,k] x_i
        ax = 2 - d
        Y = np.moveaxis(np.tensordot(A, np.moveaxis(X, ax, 0), axes=(1, 0)), 0, ax)
        if scale:
            n1 = Y.shape[2]
            s = (lam[0][None, None, :n1] + lam[1][row_lo:row_lo + ny][None, :, None]) + lam[2][:nz][:, None, None]
            Y = Y * (1.0 / (s + fd.sigma))
        return torch.from_numpy(np.ascontiguousarray(Y).ravel())
    return op


def _worker(rank, world, port, p, n_el, checks, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        kv, rules, C, A = _problem(p, n_el)
        n = [r.kv.nfun - 2 for r in rules]
        plane = n[0] * n[1]
        part = SlabPartition(n_el, p, n[2], world).validate()
        lo, hi = part.owned(rank)
        res = {}
        if "matvec" in checks:
            x = np.random.default_rng(0).standard_normal(A.N)
            dA = DistStiffness(part, plane, oracle_slab_apply(rules, C, part, rank))
            y = dA.apply(torch.from_numpy(x[lo * plane:hi * plane].copy()))
            ref = A.apply(x)[lo * plane:hi * plane]
            res["matvec"] = float(np.linalg.norm(y.numpy() - ref) / max(np.linalg.norm(ref), 1e-300))
        if "fd" in checks or "pcg" in checks:
            fd = O.FD([kv] * 3)
            dP = DistFD(part, n[0], n[1], n[2], oracle_dir_op(fd))
        if "fd" in checks:
            x = np.random.default_rng(1).standard_normal(A.N)
            z = dP.apply(torch.from_numpy(x[lo * plane:hi * plane].copy()))
            ref = fd.apply(x)[lo * plane:hi * plane]
            res["fd"] = float(np.linalg.norm(z.numpy() - ref) / np.linalg.norm(ref))
        if "pcg" in checks:
            dA = DistStiffness(part, plane, oracle_slab_apply(rules, C, part, rank))
            b = np.random.default_rng(1).standard_normal(A.N)
            u, rep = dist_cg(dA.apply, torch.from_numpy(b[lo * plane:hi * plane].copy()), dP.apply, tol=1e-8)
            uref, it, hist, *_ = O.pcg(A.apply, b, fd.apply, tol=1e-8)
            res["pcg_iters"] = (rep.iterations, it)
            res["pcg_u"] = float(np.linalg.norm(u.numpy() - uref[lo * plane:hi * plane]) /
                                 np.linalg.norm(uref[lo * plane:hi * plane]))
        out[rank] = res
    finally:
        dist.destroy_process_group()


def _run(world, p, n_el, checks):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), p, n_el, checks, out), nprocs=world, join=True)
    return dict(out)


def test_partition_windows():
    part = SlabPartition(16, 4, 18, 4).validate()
    covered = []
    for r in range(4):
        lo, hi = part.owned(r)
        covered += list(range(lo, hi))
        vlo, vhi = part.in_window(r)
        ylo, yhi = part.out_window(r)
        assert vlo == lo and hi - lo >= 1
        assert ylo == max(lo - 1, 0) and yhi == vhi  # 1 row down, p rows up
    assert covered == list(range(18))
    with pytest.raises(ValueError):
        SlabPartition(2, 3, 3, 4).validate()


@pytest.mark.parametrize("world,p,n_el", [(2, 3, 8), (3, 2, 8)])
def test_dist_matvec_matches_global(world, p, n_el):
    res = _run(world, p, n_el, ("matvec",))
    for r in range(world):
        assert res[r]["matvec"] <= 1e-13, res


def test_dist_fd_and_pcg_match_global():
    res = _run(2, 3, 8, ("fd", "pcg"))
    for r in range(2):
        assert res[r]["fd"] <= 1e-12, res
        it, it_ref = res[r]["pcg_iters"]
        assert abs(it - it_ref) <= 1, res
        assert res[r]["pcg_u"] <= 1e-9, res
