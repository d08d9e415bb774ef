"""Time the cfg-3 FD-PCG pieces: matvec, FD apply, full solve (device loop)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_08565_b200 as M
p, n_el = int(sys.argv[1]) if len(sys.argv) > 1 else 4, int(sys.argv[2]) if len(sys.argv) > 2 else 256
space = M.tensor_space(p, n_el)
A = M.setup_stiffness(space, M.build_tensor_rule(space), M.quarter_ring_map())
P = M.FDPreconditioner(space)
b = torch.from_numpy(np.random.default_rng(1).standard_normal(space.n_dofs)).cuda()
y = torch.empty_like(b)
def t(f, reps=3):
    f(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): f()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
print(f"matvec {t(lambda: A.apply(b, out=y)):.2f} ms  fd {t(lambda: P.apply(b, out=y)):.2f} ms")
t0 = time.perf_counter(); u, rep = M.cg(A.apply, b, P.apply, tol=1e-8); torch.cuda.synchronize()
print(f"pcg {time.perf_counter() - t0:.3f} s, iters {rep.iterations}")
