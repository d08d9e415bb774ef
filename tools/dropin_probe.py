"""Where the drop-in numpy apply spends its time (cfg2 p=4): fresh-output page faults, host memcpy,
pageable copies, the native pageable pipeline.  python tools/dropin_probe.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_08565_b200 as M  # noqa: E402


def t(f, n=10):
    f()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    return 1e3 * sorted(ts)[n // 2]


space = M.tensor_space(4, 128)
A = M.setup_stiffness(space, M.build_tensor_rule(space), M.identity_map(3))
N = space.n_dofs
x = np.random.default_rng(0).standard_normal(N)
y = np.empty(N)
xd = torch.from_numpy(x).cuda()
print(f"N={N} ({8 * N / 1e6:.1f} MB)")
print("fresh np.empty + first touch  ms", t(lambda: np.empty(N).fill(0.0)))
print("np.copyto (warm dst)          ms", t(lambda: np.copyto(y, x)))
print("pageable H2D (torch)          ms", t(lambda: (torch.from_numpy(x).cuda(), torch.cuda.synchronize())))
print("pageable D2H (torch)          ms", t(lambda: xd.cpu()))
print("kernel only                   ms", t(lambda: (A.apply(xd), torch.cuda.synchronize())))
print("A.apply(numpy) native pipe    ms", t(lambda: A.apply(x)))

# the bench's drop-in figure: the cfg2 sweep, numpy in / numpy out, host wall clock
ops = {}
for p in (2, 3, 4, 5, 6):
    sp = M.tensor_space(p, 128)
    ops[p] = (M.setup_stiffness(sp, M.build_tensor_rule(sp), M.identity_map(3)),
              np.random.default_rng(0).standard_normal(sp.n_dofs))
for p, (Ap, xp) in ops.items():
    print(f"p={p} A.apply(numpy) ms", t(lambda: Ap.apply(xp)))
dofs = sum(v[1].size for v in ops.values())
sweep = t(lambda: [Ap.apply(xp) for Ap, xp in ops.values()], n=10)
print(f"sweep ms {sweep:.2f}  -> {dofs / (sweep * 1e-3):.3e} DoF/s")
