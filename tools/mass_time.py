"""Mass operator timing at the cfg-3 size (quarter ring, p = 4, n_el = 256): the fused one-term kernel
against the composed K1 path (median of 10, CUDA events), with the HBM roofline of 8 (2N + Nq) bytes.
    python tools/mass_time.py [--p 4] [--n-el 256]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1712_08565_b200 as M  # noqa: E402
from paper_1712_08565_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--p", type=int, default=4)
ap.add_argument("--n-el", type=int, default=256)
a = ap.parse_args()
space = M.tensor_space(a.p, a.n_el)
Mo = M.setup_mass(space, M.build_tensor_rule(space), M.quarter_ring_map(), alpha=1.0)
x = torch.from_numpy(np.random.default_rng(0).standard_normal(space.n_dofs)).cuda()
y = torch.empty_like(x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
out = {"config": f"mass, quarter ring p={a.p} n_el={a.n_el}", "N": space.n_dofs, "Nq": Mo.n_points}
for name, path in (("fused", 0), ("composed", 1)):
    _lib.check(_lib.lib().mfwq_stiffness_set_path(Mo._h, path))
    Mo.apply(x, out=y)
    ts = []
    for _ in range(10):
        e0.record()
        Mo.apply(x, out=y)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    t = sorted(ts)[len(ts) // 2]
    nbytes = 8 * (2 * space.n_dofs + Mo.n_points)
    out[name] = {"us": t * 1e6, "achieved_gbs": nbytes / t / 1e9, "hbm_frac": nbytes / t / 1e9 / bench.peaks()["hbm_gbs"],
                 "norm": float(y.norm())}
print(json.dumps(out))
