"""BASELINE configs[0] (cfg 1): p=3, n_el=16 unit cube, one MF-WQ matvec on x = default_rng(0) and
FD-PCG to 1e-8 on the cube-sine load vector, on the GPU (public API, device tensors) and with the
CPU oracle on the host (reference algorithm), both timed; prints one JSON object."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_08565_b200 as M  # noqa: E402
from oracle import mfwq_oracle as O  # noqa: E402  (CPU arm only)

p, n_el = 3, 16
space = M.tensor_space(p, n_el)
geom = M.identity_map(3)
A = M.setup_stiffness(space, M.build_tensor_rule(space), geom)
P = M.FDPreconditioner(space)
x = torch.from_numpy(np.random.default_rng(0).standard_normal(space.n_dofs)).cuda()
b = M.assemble_rhs(space, geom, M.cube_sine_case().f)
bt = torch.as_tensor(b).cuda() if not torch.is_tensor(b) else b.cuda()
y = torch.empty_like(x)
for _ in range(5):
    A.apply(x, out=y)
    u, rep = M.cg(A.apply, bt, P.apply, tol=1e-8)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(100):
    A.apply(x, out=y)
e.record()
torch.cuda.synchronize()
mv_us = s.elapsed_time(e) * 10.0
t0 = time.perf_counter()
for _ in range(20):
    u, rep = M.cg(A.apply, bt, P.apply, tol=1e-8)
torch.cuda.synchronize()
pcg_us = (time.perf_counter() - t0) / 20 * 1e6
# CPU oracle, same inputs
rules, Aref = O.build_problem(p, n_el, "identity")
xh = x.cpu().numpy()
t0 = time.perf_counter()
for _ in range(20):
    yref = Aref.apply(xh)
cpu_mv_us = (time.perf_counter() - t0) / 20 * 1e6
Pref = O.FD([O.uniform_knots(p, n_el)] * 3)
bh = bt.cpu().numpy()
t0 = time.perf_counter()
uref, it, *_ = O.pcg(Aref.apply, bh, Pref.apply, tol=1e-8)
cpu_pcg_us = (time.perf_counter() - t0) * 1e6
print(json.dumps({"config": "cfg1 unit cube p=3 n_el=16 (N=4913)", "matvec_us": mv_us, "matvec_norm": float(y.norm()),
                  "matvec_norm_anchor": 2.41789991132909421, "pcg_us_wall": pcg_us, "pcg_iterations": rep.iterations,
                  "u_norm": float(torch.linalg.vector_norm(u)), "u_norm_anchor": 23.1045618656057385,
                  "cpu_oracle": {"matvec_us": cpu_mv_us, "pcg_us": cpu_pcg_us, "pcg_iterations": it, "cores": 1},
                  "matvec_rel_err_vs_oracle": float(np.linalg.norm(y.cpu().numpy() - yref) / np.linalg.norm(yref)),
                  "note": "launch-latency bound at this size (one fused kernel + zero pass per apply)"}))
