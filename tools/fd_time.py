"""FD apply timing (median of N, CUDA events): python tools/fd_time.py --p 4 --n-el 256 [--reps 20]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_08565_b200 as M  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--p", type=int, default=4)
ap.add_argument("--n-el", type=int, default=256)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
space = M.tensor_space(a.p, a.n_el)
P = M.FDPreconditioner(space)
x = torch.from_numpy(np.random.default_rng(0).standard_normal(space.n_dofs)).cuda()
y = torch.empty_like(x)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3):
    P.apply(x, out=y)
ts = []
for _ in range(a.reps):
    s.record()
    P.apply(x, out=y)
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e) * 1e3)
ts.sort()
n = space.n_per_dir[0]
flops = 12 * n ** 4 + space.n_dofs
med = ts[len(ts) // 2]
print(f"fd p={a.p} n_el={a.n_el} n={n}: {med:.1f} us (min {ts[0]:.1f})  {flops / med / 1e6:.2f} TF/s  "
      f"|y|={float(y.norm()):.12e}")
