"""Deterministic vs atomic accumulation of the fused matvec: median of 20 applies (CUDA events).
    python tools/det_time.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_08565_b200 as M  # noqa: E402

e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for p, n_el, geom in [(2, 128, "id"), (3, 128, "id"), (4, 128, "id"), (5, 128, "id"), (6, 128, "id"), (4, 256, "ring")]:
    space = M.tensor_space(p, n_el)
    A = M.setup_stiffness(space, M.build_tensor_rule(space), M.identity_map(3) if geom == "id" else M.quarter_ring_map())
    x = torch.from_numpy(np.random.default_rng(0).standard_normal(space.n_dofs)).cuda()
    y = torch.empty_like(x)
    res = {}
    for det in (False, True):
        A.set_deterministic(det)
        for _ in range(3):
            A.apply(x, out=y)
        ts = []
        for _ in range(20):
            e0.record()
            A.apply(x, out=y)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        res[det] = sorted(ts)[10]
    print(f"p={p} n_el={n_el} {geom}: atomics {res[False]:.1f} us  deterministic {res[True]:.1f} us "
          f"({res[True] / res[False]:.3f}x)", flush=True)
