"""cfg-3 BiCGStab (FD right-preconditioned, stored coefficients) on one GPU: iterations and time.
    python tools/profile_bicgstab.py [p] [n_el]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_08565_b200 as M  # noqa: E402

p, n_el = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (4, 256)
space = M.tensor_space(p, n_el)
A = M.setup_stiffness(space, M.build_tensor_rule(space), M.quarter_ring_map())
P = M.FDPreconditioner(space)
b = torch.from_numpy(np.random.default_rng(1).standard_normal(space.n_dofs)).cuda()
M.bicgstab(A.apply, b, P.apply, tol=1e-8, maxit=2)  # warm-up
for name, f in (("pcg", M.cg), ("bicgstab", M.bicgstab)):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    u, rep = f(A.apply, b, P.apply, tol=1e-8)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{name} p={p} n_el={n_el} N={space.n_dofs}: {rep.iterations} iterations, {dt:.4f} s wall, "
          f"matvecs {rep.matvecs}, precond {rep.precond_applies}, final {rep.residuals[-1]:.3e}, "
          f"|u|={float(torch.linalg.vector_norm(u)):.10e}")
