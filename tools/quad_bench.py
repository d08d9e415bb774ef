"""Time the device load vector and H1 error (csrc/quadrature.cu) at BASELINE sizes, with the oracle's
CPU time on cfg 1 beside it.  Prints one JSON line.

    python tools/quad_bench.py
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1712_08565_b200 as M  # noqa: E402
from oracle import mfwq_oracle as O  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e-3)
    return sorted(ts)[len(ts) // 2]


out = {"what": "device tensor-Gauss quadrature: assemble_rhs (p+1 points/span) and h1_relative_error (p+2)"}
for name, p, n_el, geom, case in [("cfg1", 3, 16, M.identity_map(3), M.cube_sine_case()),
                                  ("cfg3", 4, 256, M.quarter_ring_map(), M.oscillating_case())]:
    space = M.tensor_space(p, n_el)
    rhs = torch.empty(space.n_dofs, dtype=torch.float64, device="cuda")
    t_rhs = timed(lambda: M.assemble_rhs(space, geom, case.f, out=rhs))
    u = torch.randn(space.n_dofs, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(0)) * 1e-3
    t_h1 = timed(lambda: M.h1_relative_error(space, geom, u, case))
    npts_rhs = (n_el * (p + 1)) ** 3
    npts_err = (n_el * (p + 2)) ** 3
    out[name] = {"p": p, "n_el": n_el, "N": space.n_dofs, "rhs_s": t_rhs, "rhs_gauss_points_per_s": npts_rhs / t_rhs,
                 "h1_s": t_h1, "h1_gauss_points_per_s": npts_err / t_h1}
# CPU oracle on cfg 1 (unchunked numpy/scipy sum factorisation, one host core for the sparse part)
kv = O.uniform_knots(3, 16)
ou, og, of = O.cube_sine()
t0 = time.perf_counter()
rhs_o = O.assemble_rhs([kv] * 3, lambda xi: xi.copy(), O.jac_identity, of)
t1 = time.perf_counter()
O.error_integrals([kv] * 3, lambda xi: xi.copy(), O.jac_identity, rhs_o * 0, ou, og, 5, True)
t2 = time.perf_counter()
out["cfg1_cpu_oracle"] = {"rhs_s": t1 - t0, "h1_s": t2 - t1, "cores": 1}
print(json.dumps(out))
