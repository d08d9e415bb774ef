"""Small driver for ncu captures: builds one cfg-2/3 operator and applies it a few times.

    python tools/profile_matvec.py --p 4 --n-el 128 --geom identity --reps 3 [--fd 1]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_08565_b200 as M  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--p", type=int, default=4)
ap.add_argument("--n-el", type=int, default=128)
ap.add_argument("--geom", default="identity")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--fd", type=int, default=0)
ap.add_argument("--path", default="auto")
ap.add_argument("--otf", type=int, default=0)
a = ap.parse_args()
space = M.tensor_space(a.p, a.n_el)
A = M.setup_stiffness(space, M.build_tensor_rule(space),
                      M.identity_map(3) if a.geom == "identity" else M.quarter_ring_map(), on_the_fly=bool(a.otf))
A.set_path(a.path)
x = torch.from_numpy(np.random.default_rng(0).standard_normal(space.n_dofs)).cuda()
y = torch.empty_like(x)
P = M.FDPreconditioner(space) if a.fd else None
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for r in range(a.reps):
    s.record()
    A.apply(x, out=y)
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e) * 1e3)
    if P is not None:
        s.record()
        P.apply(x, out=y)
        e.record()
        torch.cuda.synchronize()
        print(f"fd apply: {s.elapsed_time(e)*1e3:.1f} us")
A.apply(x, out=y)
ts.sort()
print(f"matvec p={a.p} n_el={a.n_el} {a.geom}: {ts[len(ts) // 2]:.1f} us (median of {len(ts)}, min {ts[0]:.1f})"
      f"  |y|={float(y.norm()):.10e}")
