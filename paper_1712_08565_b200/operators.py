"""Matrix-free WQ stiffness operator on B200 (mirrors operators.py).

``setup_stiffness(space, rule, geom, K=None)`` returns an object whose
``apply(v, meter=None)`` runs the MF-WQ matvec (Algorithm 2,
operators.py:185-204) in hand-written sm_100a kernels through the C-ABI
(include/mfwq.h).  ``rule`` may be this package's ``TensorRule`` or the
reference's own (duck-typed: ``rules[l].weights[(a,b)]``,
``rules[l].colloc[b]``, ``rules[l].points``, ``rules[l].kv``).
"""

import ctypes as C

import numpy as np
import scipy.sparse as sp

from . import _dev, _lib
from .errors import DegenerateGeometryError  # noqa: F401  (re-export)
from .geometry import device_kind
from .kron import CostMeter, tensor_grid

#: nominal flop charge per coefficient value (operators.py:19-22)
COEFF_EVAL_FLOPS = 60

_KEYS = ((0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2))


def _csr(A):
    A = sp.csr_matrix(A)
    return (np.ascontiguousarray(A.indptr, dtype=np.int32), np.ascontiguousarray(A.indices, dtype=np.int32),
            np.ascontiguousarray(A.data, dtype=float))


def _create_handle(rule, n_dofs):
    """Library handle holding the rule's 1D factors (operators.py:146-160 restrictions done natively)."""
    L = _lib.lib()
    keep = []
    desc = _lib.StiffnessDesc()
    for l, r in enumerate(rule.rules):
        kv = r.kv
        knots = np.ascontiguousarray(kv.knots, dtype=float)
        pts = np.ascontiguousarray(r.points, dtype=float)
        keep += [knots, pts]
        desc.p[l] = int(kv.degree)
        desc.nknots[l] = len(knots)
        desc.knots[l] = _lib.dptr(knots)
        desc.npts[l] = len(pts)
        desc.pts[l] = _lib.dptr(pts)
        mats = [r.weights[(0, 0)], r.weights[(0, 1)], r.weights[(1, 0)], r.weights[(1, 1)],
                r.colloc[0], r.colloc[1]]
        for k, M in enumerate(mats):
            ip, ix, dv = _csr(M)
            keep += [ip, ix, dv]
            desc.indptr[6 * l + k] = _lib.iptr(ip)
            desc.indices[6 * l + k] = _lib.iptr(ix)
            desc.data[6 * l + k] = _lib.dptr(dv)
    h = C.c_void_p()
    _lib.check(L.mfwq_stiffness_create(C.byref(desc), C.byref(h)))
    n3 = np.zeros(3, np.int32)
    m3 = np.zeros(3, np.int32)
    N, Nq = C.c_longlong(), C.c_longlong()
    _lib.check(L.mfwq_stiffness_sizes(h, _lib.iptr(n3), _lib.iptr(m3), C.byref(N), C.byref(Nq)))
    if N.value != n_dofs:
        L.mfwq_stiffness_destroy(h)
        raise ValueError("rule and space disagree on the number of DoFs")
    return h, tuple(int(v) for v in n3), tuple(int(v) for v in m3), Nq.value



_COPY_STREAMS = {}  # device -> (H2D stream, D2H stream) for the pinned-host apply paths
_JOIN_STREAMS = {}  # device -> stream that only waits for host-pipeline D2H copies (completion events)

class StiffnessOperator:
    """Matrix-free weighted-quadrature stiffness operator (interior space)."""

    def __init__(self, space, rule, geom, K=None, on_the_fly=False, _slab=None):
        _dev.require_cuda()
        if getattr(space, "dim", 3) != 3 or len(rule.rules) != 3:
            raise NotImplementedError("the B200 operator is three-dimensional")
        self._h = None
        self.space, self.rule, self.geom, self.K = space, rule, geom, K
        self.on_the_fly = bool(on_the_fly)
        self.d = 3
        self.n_dofs = int(np.prod(space.n_per_dir))
        L = _lib.lib()
        h, self.n, self.m, self.n_points = _create_handle(rule, self.n_dofs)
        self._h = h
        # multi-GPU slab of z-elements (paper_1712_08565_b200.dist); None = whole domain
        self.slab = None
        self._in_len = self._out_len = self.n_dofs
        if _slab is not None:
            _lib.check(L.mfwq_stiffness_set_slab(h, int(_slab[0]), int(_slab[1])))
            info = np.zeros(6, np.int32)
            _lib.check(L.mfwq_stiffness_slab_info(h, _lib.iptr(info)))
            self.slab = dict(e_lo=int(info[0]), e_hi=int(info[1]), v_lo=int(info[2]), v_hi=int(info[3]),
                             y_lo=int(info[4]), y_hi=int(info[5]))
            plane = self.n[0] * self.n[1]
            self._in_len = (self.slab["v_hi"] - self.slab["v_lo"]) * plane
            self._out_len = (self.slab["y_hi"] - self.slab["y_lo"]) * plane
        if self.on_the_fly:
            self._set_on_the_fly(geom, K)
        else:
            self._set_geometry(geom, K)
        self._count_flops()

    def _count_flops(self):
        L = _lib.lib()
        fl = C.c_longlong()
        _lib.check(L.mfwq_stiffness_flops(self._h, C.byref(fl)))
        # on the fly, the reference charges one coefficient evaluation per (a, b) and apply
        # (operators.py:195-198); stored grids are charged once at setup (operators.py:162-163)
        fly = 9 * COEFF_EVAL_FLOPS * self.n_points if self.on_the_fly else 0
        self.apply_flops = fl.value + fly
        _lib.check(L.mfwq_stiffness_flops_active(self._h, C.byref(fl)))
        self.apply_flops_active = fl.value + fly  # terms with a non-zero coefficient (what runs)
        self.kernel_flops = fl.value  # the same without the reference's nominal coefficient charges
        self.setup_flops = 0 if self.on_the_fly else COEFF_EVAL_FLOPS * self.n_points * 6

    def _set_on_the_fly(self, geom, K):
        """Coefficients evaluated inside the kernel from C(xi1) (analytic maps only)."""
        kind, A = device_kind(geom)
        if kind == 3:
            raise NotImplementedError("on-the-fly coefficients need an analytic map (identity, affine or "
                                      "quarter ring); use stored grids for general geometries")
        K9 = None
        if K is not None:
            Ka = None if callable(K) else np.asarray(K, dtype=float)
            if Ka is None or Ka.shape != (3, 3):
                raise NotImplementedError("on-the-fly coefficients take K = None or a constant 3x3 K")
            K9 = np.ascontiguousarray(Ka)
        _lib.check(_lib.lib().mfwq_stiffness_set_on_the_fly(
            self._h, kind, _lib.dptr(A) if A is not None else None, _lib.dptr(K9) if K9 is not None else None,
            C.c_void_p(_dev.stream_ptr())))

    def set_on_the_fly(self, enabled: bool):
        """Switch between stored grids and on-the-fly evaluation (operators.py:171-176)."""
        enabled = bool(enabled)
        if enabled and not self.on_the_fly:
            self._set_on_the_fly(self.geom, self.K)
        elif not enabled and self.on_the_fly:
            self._set_geometry(self.geom, self.K)
        self.on_the_fly = enabled
        self._count_flops()

    # -- coefficient grids (operators.py:64-84) --------------------------------
    def _points(self):
        return np.stack(tensor_grid([r.points for r in self.rule.rules]), axis=1)

    def _set_geometry(self, geom, K):
        L = _lib.lib()
        s = C.c_void_p(_dev.stream_ptr())
        kind, A = device_kind(geom)
        K9 = None
        Kfield = None
        if K is not None:
            if callable(K):
                xi = self._points()
                Kfield = _dev.to_device(np.asarray(K(geom.evaluate(xi)), dtype=float).reshape(-1))[0]
            else:
                Ka = np.asarray(K, dtype=float)
                if Ka.shape == (3, 3):
                    K9 = np.ascontiguousarray(Ka)
                else:
                    Kfield = _dev.to_device(Ka.reshape(-1))[0]
        J = None
        if kind == 3:
            xi = self._points()
            J = _dev.to_device(np.asarray(geom.jacobian(xi), dtype=float).reshape(-1))[0]
        rc = L.mfwq_stiffness_set_geometry(
            self._h, kind, _lib.dptr(A) if A is not None else None, _lib.dptr(K9) if K9 is not None else None,
            C.c_void_p(J.data_ptr()) if J is not None else None,
            C.c_void_p(Kfield.data_ptr()) if Kfield is not None else None, s)
        _lib.check(rc)

    @property
    def coeff_scalars(self) -> int:
        return 0 if self.on_the_fly else 6 * self.n_points

    @property
    def coeffs(self):
        """The six symmetric grids keyed (a<=b) as host arrays (operators.py:84); None on the fly."""
        if self.on_the_fly:
            return None
        out = {}
        for k, key in enumerate(_KEYS):
            g = _dev.empty(self.n_points)
            _lib.check(_lib.lib().mfwq_stiffness_get_coeff(self._h, k, C.c_void_p(g.data_ptr()),
                                                           C.c_void_p(_dev.stream_ptr())))
            out[key] = g.cpu().numpy()
        return out

    def set_path(self, path: str):
        """'auto' | 'generic' | 'fused' kernel path (all on the GPU)."""
        _lib.check(_lib.lib().mfwq_stiffness_set_path(self._h, {"auto": 0, "generic": 1, "fused": 2}[path]))

    def set_deterministic(self, enabled: bool = True):
        """Bitwise reproducible applies: the fused kernel's overlapping output windows are summed
        in a fixed order instead of by fp64 atomics (the reference's numpy apply is deterministic)."""
        self.deterministic = bool(enabled)
        _lib.check(_lib.lib().mfwq_stiffness_set_deterministic(self._h, int(self.deterministic)))

    def info(self):
        tm, ok, nt = C.c_int(), C.c_int(), C.c_int()
        _lib.check(_lib.lib().mfwq_stiffness_info(self._h, C.byref(tm), C.byref(ok), C.byref(nt)))
        return {"term_mask": tm.value, "fused_ok": bool(ok.value), "kernel_terms": nt.value}

    # -- apply (operators.py:185-204) -----------------------------------------
    def apply(self, v, meter: CostMeter | None = None, out=None):
        if _dev.is_pinned_host(v):
            return self._apply_pinned(v, meter, out)
        if out is None and isinstance(v, np.ndarray):
            return self._apply_numpy(v, meter)
        x, host = _dev.to_device(v, self._in_len)
        y = _dev.check_out(out, self._out_len) if out is not None else _dev.empty(self._out_len)
        _lib.check(_lib.lib().mfwq_stiffness_apply(self._h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()),
                                                   C.c_void_p(_dev.stream_ptr())))
        if meter is not None:
            meter.add_flops(self.apply_flops)
        return _dev.back(y, host)

    __call__ = apply

    def _apply_numpy(self, v, meter):
        """numpy in, fresh numpy out (operators.py:185-189 semantics): the native pageable pipeline
        (mfwq_stiffness_apply_pageable) stages both vectors through pinned chunks on host threads."""
        x = np.ascontiguousarray(np.asarray(v, dtype=float).ravel())
        if x.size != self._in_len:
            raise ValueError(f"expected vector of length {self._in_len}, got {x.size}")
        y = np.empty(self._out_len)
        _lib.check(_lib.lib().mfwq_stiffness_apply_pageable(self._h, C.c_void_p(x.ctypes.data),
                                                            C.c_void_p(y.ctypes.data),
                                                            C.c_void_p(_dev.stream_ptr())))
        if meter is not None:
            meter.add_flops(self.apply_flops)
        return y

    def apply_pipelined(self, v, out=None, meter: CostMeter | None = None):
        """Streaming form of ``apply`` for pinned host tensors: H2D on one side stream, the kernel on
        the current stream, D2H on another side stream, two staging buffers.  A sequence of calls keeps
        both copy directions and the SMs busy at once.  Returns ``(out, event)``; ``out`` is valid once
        ``event`` has completed (``event.synchronize()`` or ``torch.cuda.synchronize()``)."""
        if not _dev.is_pinned_host(v):
            raise ValueError("apply_pipelined takes a pinned host torch tensor")
        torch = _dev.torch
        if v.numel() != self._in_len:
            raise ValueError(f"expected vector of length {self._in_len}, got {v.numel()}")
        o = out if out is not None else torch.empty(self._out_len, dtype=torch.float64, pin_memory=True)
        if o.numel() != self._out_len or o.is_cuda or o.dtype != torch.float64 or not o.is_contiguous():
            raise ValueError("out must be a contiguous float64 host tensor of the output length")
        x = v.reshape(-1)
        if x.dtype != torch.float64 or not x.is_contiguous():
            # a converted temporary could be recycled by torch's pinned allocator while the raw copy
            # that reads it is still queued: the caller owns (and keeps alive) the input buffer
            raise ValueError("apply_pipelined takes a contiguous float64 pinned host tensor")
        cur = torch.cuda.current_stream()
        # native pipeline (mfwq_stiffness_apply_host): H2D / kernel / D2H on three streams, two device
        # staging pairs per operator; no per-call Python stream or event objects
        _lib.check(_lib.lib().mfwq_stiffness_apply_host(self._h, C.c_void_p(x.data_ptr()), C.c_void_p(o.data_ptr()),
                                                        C.c_void_p(cur.cuda_stream)))
        dev = torch.cuda.current_device()
        if dev not in _JOIN_STREAMS:
            _JOIN_STREAMS[dev] = torch.cuda.Stream()
        js = _JOIN_STREAMS[dev]
        _lib.check(_lib.lib().mfwq_stiffness_host_join(self._h, C.c_void_p(js.cuda_stream)))
        done = torch.cuda.Event()
        done.record(js)
        self._host_keep = (x, o)  # host buffers stay referenced while their copies are in flight
        if meter is not None:
            meter.add_flops(self.apply_flops)
        return o, done

    def _apply_pinned(self, v, meter, out, d2h_side=False):
        """Pinned host torch tensor in, pinned host tensor out, asynchronous like torch's non_blocking
        copies: with d2h_side=False the result is valid once the current stream is synchronised.  The
        input copy runs on a side stream into one of two device staging buffers, so consecutive calls
        overlap the H2D of call k+1 with the kernel and the D2H of call k."""
        torch = _dev.torch
        if v.numel() != self._in_len:
            raise ValueError(f"expected vector of length {self._in_len}, got {v.numel()}")
        st = getattr(self, "_pipe", None)
        if st is None:
            # one H2D and one D2H side stream per device, shared by all operators: consecutive calls on
            # different operators then form a single in-order copy pipeline in each direction
            dev = torch.cuda.current_device()
            if dev not in _COPY_STREAMS:
                _COPY_STREAMS[dev] = (torch.cuda.Stream(), torch.cuda.Stream())
            h2d_s, d2h_s = _COPY_STREAMS[dev]
            st = self._pipe = {"h2d": h2d_s, "d2h": d2h_s,
                               "x": [_dev.empty(self._in_len) for _ in range(2)],
                               "y": [_dev.empty(self._out_len) for _ in range(2)], "free": [None, None],
                               "read": [None, None], "i": 0}
        i = st["i"]
        st["i"] ^= 1
        cur = torch.cuda.current_stream()
        h2d = st["h2d"]
        if st["free"][i] is not None:
            h2d.wait_event(st["free"][i])  # the kernel that last read this staging buffer is done
        with torch.cuda.stream(h2d):
            st["x"][i].copy_(v.reshape(-1).to(torch.float64), non_blocking=True)
            landed = torch.cuda.Event()
            landed.record(h2d)
        cur.wait_event(landed)
        if st["read"][i] is not None:
            cur.wait_event(st["read"][i])  # the side-stream D2H that last read this staging buffer is done
        _lib.check(_lib.lib().mfwq_stiffness_apply(self._h, C.c_void_p(st["x"][i].data_ptr()),
                                                   C.c_void_p(st["y"][i].data_ptr()), C.c_void_p(cur.cuda_stream)))
        free = torch.cuda.Event()
        free.record(cur)
        st["free"][i] = free
        o = out if out is not None else torch.empty(self._out_len, dtype=torch.float64, pin_memory=True)
        if o.numel() != self._out_len or o.is_cuda:
            raise ValueError("out must be a host tensor of the output length")
        if meter is not None:
            meter.add_flops(self.apply_flops)
        if not d2h_side:
            o.reshape(-1).copy_(st["y"][i], non_blocking=True)
            st["read"][i] = None
            return o
        d2h = st["d2h"]
        d2h.wait_event(free)
        with torch.cuda.stream(d2h):
            o.reshape(-1).copy_(st["y"][i], non_blocking=True)
            done = torch.cuda.Event()
            done.record(d2h)
        st["read"][i] = done
        return o, done

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            _lib._lib.mfwq_stiffness_destroy(h)
            self._h = None


def setup_stiffness(space, rule, geom, K=None, on_the_fly=False) -> StiffnessOperator:
    """operators.py:227-228."""
    return StiffnessOperator(space, rule, geom, K=K, on_the_fly=on_the_fly)


class MassOperator:
    """Matrix-free weighted-quadrature mass operator on the interior space (operators.py:87-132).

    w = (W00 x W00 x W00)(alpha det J o (B0 x B0 x B0) v), composed on the GPU from the banded
    one-mode contraction kernels; the alpha det J grid is built on the device (operators.py:46-61)
    or, on the fly, for every apply.
    """

    def __init__(self, space, rule, geom, alpha=1.0, on_the_fly=False):
        _dev.require_cuda()
        if getattr(space, "dim", 3) != 3 or len(rule.rules) != 3:
            raise NotImplementedError("the B200 operator is three-dimensional")
        self._h = None
        self.space, self.rule, self.geom, self.alpha = space, rule, geom, alpha
        self.on_the_fly = bool(on_the_fly)
        self.n_dofs = int(np.prod(space.n_per_dir))
        self.n = tuple(space.n_per_dir)
        self._h, _, _, self.n_points = _create_handle(rule, self.n_dofs)
        self._afield = None
        if callable(alpha):
            xi = np.stack(tensor_grid([r.points for r in rule.rules]), axis=1)
            self._afield = _dev.to_device(np.asarray(alpha(geom.evaluate(xi)), dtype=float).reshape(-1),
                                          self.n_points)[0]
        self._set(self.on_the_fly)

    def _set(self, fly):
        kind, A = device_kind(self.geom)
        J = None
        if kind == 3:
            if fly:
                raise NotImplementedError("on-the-fly mass coefficients need an analytic map")
            xi = np.stack(tensor_grid([r.points for r in self.rule.rules]), axis=1)
            J = _dev.to_device(np.asarray(self.geom.jacobian(xi), dtype=float).reshape(-1))[0]
        a = 1.0 if callable(self.alpha) else float(self.alpha)
        _lib.check(_lib.lib().mfwq_mass_set(
            self._h, kind, _lib.dptr(A) if A is not None else None, C.c_void_p(J.data_ptr()) if J is not None else None,
            a, C.c_void_p(self._afield.data_ptr()) if self._afield is not None else None, int(fly),
            C.c_void_p(_dev.stream_ptr())))
        fl = C.c_longlong()
        _lib.check(_lib.lib().mfwq_mass_flops(self._h, C.byref(fl)))
        self.apply_flops = fl.value + (COEFF_EVAL_FLOPS * self.n_points if fly else 0)
        self.setup_flops = 0 if fly else COEFF_EVAL_FLOPS * self.n_points

    @property
    def coeff_scalars(self) -> int:
        """Stored coefficient-grid scalars (operators.py:104-107)."""
        return 0 if self.on_the_fly else self.n_points

    def set_on_the_fly(self, enabled: bool):
        """Toggle on-the-fly coefficient evaluation (operators.py:109-115)."""
        enabled = bool(enabled)
        if enabled != self.on_the_fly:
            self._set(enabled)
        self.on_the_fly = enabled

    def apply(self, v, meter: CostMeter | None = None, out=None):
        x, host = _dev.to_device(v, self.n_dofs)
        y = _dev.check_out(out, self.n_dofs) if out is not None else _dev.empty(self.n_dofs)
        _lib.check(_lib.lib().mfwq_mass_apply(self._h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()),
                                              C.c_void_p(_dev.stream_ptr())))
        if meter is not None:
            meter.add_flops(self.apply_flops)
        return _dev.back(y, host)

    __call__ = apply

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            _lib._lib.mfwq_stiffness_destroy(h)
            self._h = None


def setup_mass(space, rule, geom, alpha=1.0, on_the_fly=False) -> MassOperator:
    """operators.py:223-224."""
    return MassOperator(space, rule, geom, alpha=alpha, on_the_fly=on_the_fly)


def apply_system(mass_op, stiff_op, v, meter: CostMeter | None = None):
    """Stiffness plus mass (operators.py:231-245); the mass term is skipped when absent or alpha == 0."""
    x, host = _dev.to_device(v, stiff_op.n_dofs)
    w = stiff_op.apply(x, meter)
    skip_mass = mass_op is None or (not callable(mass_op.alpha) and float(mass_op.alpha) == 0.0)
    if not skip_mass:
        m = mass_op.apply(x, meter)
        _lib.check(_lib.lib().mfwq_axpy(C.c_void_p(w.data_ptr()), C.c_void_p(m.data_ptr()), w.numel(), 1.0,
                                        C.c_void_p(_dev.stream_ptr())))
        if meter is not None:
            meter.add_flops(2 * stiff_op.n_dofs)
    return _dev.back(w, host)


class SystemOperator:
    """(stiffness + mass) as a single apply (operators.py:248-257)."""

    def __init__(self, stiff_op, mass_op=None):
        self.stiff_op = stiff_op
        self.mass_op = mass_op
        self.n_dofs = stiff_op.n_dofs

    def apply(self, v, meter: CostMeter | None = None):
        return apply_system(self.mass_op, self.stiff_op, v, meter)

    __call__ = apply
