import os, sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_1712_08565_b200 as M
space = M.tensor_space(3, 16); geom = M.identity_map(3)
A = M.setup_stiffness(space, M.build_tensor_rule(space), geom); P = M.FDPreconditioner(space)
b = M.assemble_rhs(space, geom, M.cube_sine_case().f); b = torch.as_tensor(b).cuda()
x = torch.empty_like(b)
def wall(f, n=50):
    for _ in range(5): f()
    torch.cuda.synchronize(); ts=[]
    for _ in range(n):
        t0=time.perf_counter(); f(); torch.cuda.synchronize(); ts.append((time.perf_counter()-t0)*1e6)
    ts.sort(); return ts[len(ts)//2]
print("matvec+sync", wall(lambda: A.apply(b, out=x)))
print("fd+sync", wall(lambda: P.apply(b, out=x)))
print("empty sync", wall(lambda: None))
print("cg graphs", wall(lambda: M.cg(A.apply, b, P.apply, tol=1e-8)))
os.environ["MFWQ_NO_PCG_GRAPHS"]="1"
print("cg eager", wall(lambda: M.cg(A.apply, b, P.apply, tol=1e-8)))
del os.environ["MFWQ_NO_PCG_GRAPHS"]
# GPU-side duration of one solve
e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
e0.record(); M.cg(A.apply, b, P.apply, tol=1e-8); e1.record(); torch.cuda.synchronize(); print("cg events", e0.elapsed_time(e1)*1e3)
