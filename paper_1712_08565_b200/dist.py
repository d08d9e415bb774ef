"""Multi-GPU slab decomposition along xi_3.

One process per GPU (torch.distributed, NCCL over NVLink; gloo on CPU for the
tests).  The tensor grid is cut into contiguous z-element slabs; because xi_3 is
the slowest index, a rank's DoF planes are a contiguous chunk of the flat vector.

* Matvec: rank r owns z-elements [E_r, E_{r+1}) and interior DoF planes
  [lo_r, hi_r) = [E_r - 1, E_{r+1} - 1) (first/last rank clipped to [0, n3)).  Its
  elements read planes [E_r - 1, E_{r+1} + p - 1)  -> forward halo: p planes from
  above; they write rows [E_r - 2, E_{r+1} + p - 1)  -> reverse halo: 1 row down,
  p rows up, added by the owners.  (Element e touches full functions e..e+p on
  the B side; its left breakpoint also closes the support of function e-1, whose
  WQ weights there are non-zero, wq.py:89.)
* FD: directions 1 and 2 are local; direction 3 is an all-to-all transpose to a
  partition of the i2 rows, the U3^T contraction with the fused eigenvalue scale,
  the U3 contraction, and the transpose back.
* PCG: the reference recurrence (solvers.py:137-173) with every dot product
  allreduced (one scalar pair per reduction).

The exchange code only needs torch tensors and a process group; local compute
is injected, so the same protocol runs with the CUDA kernels (NCCL) and with a
numpy oracle (gloo) in tests/test_dist_gloo.py.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

try:
    import torch
    import torch.distributed as dist
except ImportError:  # pragma: no cover
    torch = None
    dist = None


@dataclass(frozen=True)
class SlabPartition:
    """Element / plane ownership for `world` ranks along xi_3."""

    n_el: int
    p: int
    n3: int
    world: int

    @property
    def E(self):
        return [r * self.n_el // self.world for r in range(self.world + 1)]

    def owned(self, r):
        E = self.E
        lo = 0 if r == 0 else E[r] - 1
        hi = self.n3 if r == self.world - 1 else E[r + 1] - 1
        return lo, hi

    def elements(self, r):
        return self.E[r], self.E[r + 1]

    def in_window(self, r):  # planes read by rank r's elements
        e0, e1 = self.elements(r)
        return max(e0 - 1, 0), min(e1 + self.p - 1, self.n3)

    def out_window(self, r):  # rows written by rank r's elements
        e0, e1 = self.elements(r)
        return max(e0 - 2, 0), min(e1 + self.p - 1, self.n3)

    def validate(self):
        for r in range(self.world):
            lo, hi = self.owned(r)
            if hi <= lo or self.E[r + 1] <= self.E[r]:
                raise ValueError(f"rank {r} owns no DoF plane (n_el={self.n_el}, world={self.world})")
        return self

    def owners(self, a, b):
        """[(rank, a', b')] covering planes [a, b)."""
        out = []
        for r in range(self.world):
            lo, hi = self.owned(r)
            s, e = max(a, lo), min(b, hi)
            if s < e:
                out.append((r, s, e))
        return out

    def rows(self, s, n2):  # i2 rows of rank s in the transposed (direction-3) layout
        return s * n2 // self.world, (s + 1) * n2 // self.world


def _exchange(ops_send, ops_recv, group=None):
    """Post all sends/receives of this rank as ONE batch, then wait.

    Under NCCL the batch is a single ncclGroupStart/End, so a rank that both sends to and receives
    from the same peer (the reverse halo: p rows up, one row down) cannot deadlock on the ordering of
    separately launched send/recv kernels; gloo runs the ops one by one.  A rank with nothing to
    exchange posts nothing (never the group's first collective: dist_cg allreduces ||b|| first)."""
    ops = [dist.P2POp(dist.irecv, t, peer, group=group) for t, peer in ops_recv]
    ops += [dist.P2POp(dist.isend, t, peer, group=group) for t, peer in ops_send]
    if not ops:
        return
    for q in dist.batch_isend_irecv(ops):
        q.wait()


class DistStiffness:
    """Slab-distributed MF-WQ matvec: owned planes in, owned planes out.

    local_apply(x_window) -> y_window maps the rank's input window (planes
    part.in_window(rank)) to its output window (rows part.out_window(rank)).
    """

    def __init__(self, part: SlabPartition, plane: int, local_apply, rank=None, group=None):
        self.part, self.plane, self.local_apply, self.group = part, plane, local_apply, group
        self.rank = dist.get_rank(group) if rank is None else rank

    def apply(self, x_owned):
        P, r, pl = self.part, self.rank, self.plane
        lo, hi = P.owned(r)
        vlo, vhi = P.in_window(r)
        dev, dt = x_owned.device, x_owned.dtype
        # forward halo: planes [hi, vhi) from their owners; every rank runs the same plan
        xin = torch.empty((vhi - vlo) * pl, dtype=dt, device=dev)
        xin[(lo - vlo) * pl:(hi - vlo) * pl] = x_owned
        sends, recvs = [], []
        for q in range(P.world):
            qlo, qhi = P.owned(q)
            qvlo, qvhi = P.in_window(q)
            for (o, a, b) in P.owners(qhi, qvhi):
                if q == r and o != r:
                    recvs.append((xin[(a - vlo) * pl:(b - vlo) * pl], o))
                if o == r and q != r:
                    sends.append((x_owned[(a - lo) * pl:(b - lo) * pl].contiguous(), q))
        _exchange(sends, recvs, self.group)
        yout = self.local_apply(xin)
        ylo, yhi = P.out_window(r)
        y = yout[(lo - ylo) * pl:(hi - ylo) * pl].clone()
        # reverse halo: rows outside [lo, hi) go to their owners and are added there
        sends, recvs, adds = [], [], []
        for q in range(P.world):
            qlo, qhi = P.owned(q)
            qylo, qyhi = P.out_window(q)
            for (a, b) in ((qylo, qlo), (qhi, qyhi)):
                for (o, s, e) in P.owners(a, b):
                    if q == r and o != r:
                        sends.append((yout[(s - ylo) * pl:(e - ylo) * pl].contiguous(), o))
                    if o == r and q != r:
                        buf = torch.empty((e - s) * pl, dtype=dt, device=dev)
                        recvs.append((buf, q))
                        adds.append((buf, s))
        _exchange(sends, recvs, self.group)
        for buf, s in adds:
            y[(s - lo) * pl:(s - lo) * pl + buf.numel()] += buf
        return y


class DistFD:
    """Slab-distributed FD apply; dir_op(dir, inverse, scale, x, nz, ny, row_lo) -> y."""

    def __init__(self, part: SlabPartition, n1: int, n2: int, n3: int, dir_op, rank=None, group=None):
        self.part, self.n1, self.n2, self.n3, self.dir_op, self.group = part, n1, n2, n3, dir_op, group
        self.rank = dist.get_rank(group) if rank is None else rank

    def _to_rows(self, s2, nz):
        P, n1, n2 = self.part, self.n1, self.n2
        blocks = [s2.view(nz, n2, n1)[:, slice(*P.rows(s, n2)), :].reshape(-1) for s in range(P.world)]
        inp = torch.cat(blocks)
        r0, r1 = P.rows(self.rank, n2)
        in_splits = [b.numel() for b in blocks]
        out_splits = [(P.owned(q)[1] - P.owned(q)[0]) * (r1 - r0) * n1 for q in range(P.world)]
        out = torch.empty(sum(out_splits), dtype=s2.dtype, device=s2.device)
        dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)
        return out  # (n3, rows_mine, n1): blocks arrive in plane order

    def _from_rows(self, t, nz):
        P, n1, n2 = self.part, self.n1, self.n2
        r0, r1 = P.rows(self.rank, n2)
        tv = t.view(self.n3, r1 - r0, n1)
        blocks = [tv[slice(*P.owned(q))].reshape(-1) for q in range(P.world)]
        inp = torch.cat(blocks)
        in_splits = [b.numel() for b in blocks]
        out_splits = [nz * (P.rows(q, n2)[1] - P.rows(q, n2)[0]) * n1 for q in range(P.world)]
        out = torch.empty(sum(out_splits), dtype=t.dtype, device=t.device)
        dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)
        res = torch.empty(nz, n2, n1, dtype=t.dtype, device=t.device)
        off = 0
        for q in range(P.world):
            q0, q1 = P.rows(q, n2)
            k = nz * (q1 - q0) * n1
            res[:, q0:q1, :] = out[off:off + k].view(nz, q1 - q0, n1)
            off += k
        return res.reshape(-1)

    def apply(self, r_owned):
        lo, hi = self.part.owned(self.rank)
        nz = hi - lo
        r0, r1 = self.part.rows(self.rank, self.n2)
        s1 = self.dir_op(0, 0, 0, r_owned, nz, self.n2, 0)
        s2 = self.dir_op(1, 0, 0, s1, nz, self.n2, 0)
        t = self._to_rows(s2, nz)
        t = self.dir_op(2, 0, 1, t, self.n3, r1 - r0, r0)
        t = self.dir_op(2, 1, 0, t, self.n3, r1 - r0, r0)
        s3 = self._from_rows(t, nz)
        s4 = self.dir_op(1, 1, 0, s3, nz, self.n2, 0)
        return self.dir_op(0, 1, 0, s4, nz, self.n2, 0)


def dist_cg(apply_A, b_owned, apply_P=None, tol=1e-8, maxit=1000, group=None):
    """PCG of solvers.py:137-173 over owned slices; dots are allreduced."""
    from .solvers import IndefiniteOperatorError, KrylovReport

    def gdot(u, v):
        t = torch.stack([(u * v).sum()])
        dist.all_reduce(t, group=group)
        return float(t[0])

    x = torch.zeros_like(b_owned)
    bnorm = gdot(b_owned, b_owned) ** 0.5
    if bnorm == 0.0:
        return x, KrylovReport(0, [0.0], True, 0, 0)
    P = apply_P if apply_P is not None else (lambda v: v)
    r = b_owned.clone()
    z = P(r)
    precs, matvecs = 1, 0
    p = z.clone()
    rz = gdot(r, z)
    hist = [1.0]
    for k in range(1, maxit + 1):
        Ap = apply_A(p)
        matvecs += 1
        pAp = gdot(p, Ap)
        if pAp <= 0:
            raise IndefiniteOperatorError(f"nonpositive curvature p.Ap = {pAp:.3e} at iteration {k}")
        alpha = rz / pAp
        x += alpha * p
        r -= alpha * Ap
        rel = gdot(r, r) ** 0.5 / bnorm
        hist.append(rel)
        if rel <= tol:
            return x, KrylovReport(k, hist, True, matvecs, precs)
        z = P(r)
        precs += 1
        rz_new = gdot(r, z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, KrylovReport(maxit, hist, False, matvecs, precs)


# ---------------------------------------------------------------------------
# CUDA bindings: the local pieces run in libmfwq.so
# ---------------------------------------------------------------------------
def cuda_stiffness(space, rule, geom, part: SlabPartition, rank, K=None):
    """Local slab operator (fused sm_100a kernel restricted to the rank's z-elements)."""
    from .operators import StiffnessOperator
    op = StiffnessOperator(space, rule, geom, K=K, _slab=part.elements(rank))
    return op, (lambda xin: op.apply(xin))


def cuda_fd_dir_op(fd):
    """dir_op for DistFD backed by mfwq_fd_apply_dir."""
    from . import _dev, _lib

    def op(d, inverse, scale, x, nz, ny, row_lo):
        y = torch.empty_like(x)
        _lib.check(_lib.lib().mfwq_fd_apply_dir(fd._h, d, inverse, scale, C.c_void_p(x.data_ptr()),
                                                C.c_void_p(y.data_ptr()), nz, ny, row_lo,
                                                C.c_void_p(_dev.stream_ptr())))
        return y
    return op


# ---------------------------------------------------------------------------
# native comm-aware solver (libmfwq.so mfwq_pcg_solve_comm): halo exchanges, FD all-to-all and
# allreduced PCG scalars inside the library; one host read per iteration
# ---------------------------------------------------------------------------
def nccl_library():
    """Path of the NCCL torch bundles (the one torch.distributed itself loaded)."""
    import glob
    import os
    try:
        import nvidia.nccl as nc
        for base in nc.__path__:
            hits = sorted(glob.glob(os.path.join(base, "lib", "libnccl.so*")))
            if hits:
                return hits[0]
    except ImportError:
        pass
    raise RuntimeError("torch's bundled NCCL (nvidia.nccl) not found")


class Communicator:
    """Transport of the native slab solver: ``Communicator.local(P)`` drives all P ranks of the
    partition from this process on the current device (single-GPU emulation of the multi-GPU path:
    same solver, slab kernels and messages, one cudaMemcpyAsync per message), ``Communicator.nccl()``
    is one rank per process / GPU over NCCL (NVLink), set up from a torch.distributed group."""

    def __init__(self, handle):
        from . import _lib
        self._h = handle
        w, nl, f = C.c_int(), C.c_int(), C.c_int()
        _lib.check(_lib.lib().mfwq_comm_info(handle, C.byref(w), C.byref(nl), C.byref(f)))
        self.world, self.nlocal, self.first = w.value, nl.value, f.value

    @classmethod
    def local(cls, world):
        from . import _lib
        h = C.c_void_p()
        _lib.check(_lib.lib().mfwq_comm_create_local(int(world), C.byref(h)))
        return cls(h)

    @classmethod
    def nccl(cls, group=None):
        from . import _lib
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        lib = nccl_library().encode()
        uid = C.create_string_buffer(128)
        if rank == 0:
            _lib.check(_lib.lib().mfwq_nccl_unique_id(lib, uid))
        obj = [bytes(uid.raw) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        uid = C.create_string_buffer(obj[0], 128)
        h = C.c_void_p()
        _lib.check(_lib.lib().mfwq_comm_create_nccl(lib, uid, world, rank, C.byref(h)))
        return cls(h)

    def __del__(self):
        import sys
        h = getattr(self, "_h", None)
        if h is not None and not sys.is_finalizing():  # no NCCL teardown during interpreter exit
            from . import _lib
            if _lib._lib is not None:
                _lib._lib.mfwq_comm_destroy(h)
            self._h = None


class SlabSolver:
    """Slab-distributed FD-PCG (solvers.py:137-173) with the ranks this process drives.

    ``cg(b_slices, tol, maxit)`` takes each local rank's owned slice of b (device tensors, planes
    SlabPartition.owned(rank)) and returns (x slices, KrylovReport); the report is the global one."""

    def __init__(self, space, rule, geom, comm: Communicator, K=None, on_the_fly=False):
        from .operators import StiffnessOperator
        from .solvers import FDPreconditioner
        kv = space.knotvectors[2]
        self.n = [k.n_funcs - 2 for k in space.knotvectors]
        self.plane = self.n[0] * self.n[1]
        self.part = SlabPartition(len(np.unique(kv.knots)) - 1, kv.degree, self.n[2], comm.world).validate()
        self.comm = comm
        self.ranks = list(range(comm.first, comm.first + comm.nlocal))
        self.ops = [StiffnessOperator(space, rule, geom, K=K, on_the_fly=on_the_fly, _slab=self.part.elements(r))
                    for r in self.ranks]
        self.P = FDPreconditioner(space)

    def owned_slices(self, full):
        """The local ranks' owned slices of a full-length vector (views)."""
        return [full[slice(*(v * self.plane for v in self.part.owned(r)))] for r in self.ranks]

    def cg(self, b_slices, tol=1e-8, maxit=1000):
        from . import _dev, _lib
        from .solvers import KrylovReport
        bs = [_dev.to_device(b, (self.part.owned(r)[1] - self.part.owned(r)[0]) * self.plane)[0]
              for b, r in zip(b_slices, self.ranks)]
        xs = [torch.empty_like(b) for b in bs]
        n = len(bs)
        ops = (C.c_void_p * n)(*[op._h for op in self.ops])
        bp = (C.c_void_p * n)(*[b.data_ptr() for b in bs])
        xp = (C.c_void_p * n)(*[x.data_ptr() for x in xs])
        hist = np.zeros(maxit + 1)
        rep = _lib.KrylovReportC()
        _lib.check(_lib.lib().mfwq_pcg_solve_comm(self.comm._h, ops, self.P._h, bp, xp, float(tol), int(maxit),
                                                  _lib.dptr(hist), C.byref(rep), C.c_void_p(_dev.stream_ptr())))
        report = KrylovReport(rep.iterations, hist[:rep.n_residuals].tolist(), bool(rep.converged), rep.matvecs,
                              rep.precond_applies)
        return xs, report


def setup_distributed(space, rule, geom, K=None, group=None):
    """(DistStiffness, DistFD, partition) for this rank, on its CUDA device."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    kv = space.knotvectors[2]
    n = [kv_.n_funcs - 2 for kv_ in space.knotvectors]
    part = SlabPartition(len(np.unique(kv.knots)) - 1, kv.degree, n[2], world).validate()
    op, local = cuda_stiffness(space, rule, geom, part, rank, K)
    A = DistStiffness(part, n[0] * n[1], local, rank, group)
    from .solvers import FDPreconditioner
    fd = FDPreconditioner(space)
    Pd = DistFD(part, n[0], n[1], n[2], cuda_fd_dir_op(fd), rank, group)
    A._keep = (op, fd)
    return A, Pd, part
