"""Time the native slab-distributed FD-PCG with all P ranks emulated on ONE GPU (in-process transport)
against the single-GPU device PCG, at cfg 3 and cfg 5.  The emulated solve runs every rank's kernels
and messages back to back on one device, so its time is NOT a multi-GPU time: the excess over the
single-GPU solve is the distributed algorithm's own overhead (halo / all-to-all copies, packing,
per-slab launches).  Prints one JSON object.

    python tools/slab_emulation.py [--cfgs 3,5] [--worlds 2,4,8]
"""
import argparse
import gc
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_08565_b200 as M  # noqa: E402
from paper_1712_08565_b200 import _lib  # noqa: E402
from paper_1712_08565_b200.dist import Communicator, SlabSolver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfgs", default="3,5")
ap.add_argument("--worlds", default="2,4,8")
a = ap.parse_args()
CFG = {3: (4, 256), 5: (6, 512)}
out = {}


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = _lib.lib().mfwq_launch_count()
    e0.record()
    res = fn()
    e1.record()
    torch.cuda.synchronize()
    return res, e0.elapsed_time(e1) * 1e-3, _lib.lib().mfwq_launch_count() - l0


for c in [int(v) for v in a.cfgs.split(",")]:
    p, n_el = CFG[c]
    space = M.tensor_space(p, n_el)
    rule = M.build_tensor_rule(space)
    geom = M.quarter_ring_map()
    b = torch.from_numpy(np.random.default_rng(1).standard_normal(space.n_dofs)).cuda()
    A = M.setup_stiffness(space, rule, geom)
    P = M.FDPreconditioner(space)
    (u1, r1), t1, l1 = timed(lambda: M.cg(A.apply, b, P.apply, tol=1e-8))
    u1 = u1.cpu()
    del A, P
    gc.collect()
    torch.cuda.empty_cache()
    res = {"N": space.n_dofs, "single_gpu": {"iterations": r1.iterations, "solve_s": t1, "launches": l1}}
    for w in [int(v) for v in a.worlds.split(",")]:
        S = SlabSolver(space, rule, geom, Communicator.local(w))
        bs = S.owned_slices(b)
        (xs, rP), tP, lP = timed(lambda: S.cg(bs, tol=1e-8))
        d = float(torch.linalg.vector_norm(torch.cat(xs).cpu() - u1) / torch.linalg.vector_norm(u1))
        res[f"emulated_x{w}"] = {"iterations": rP.iterations, "solve_s": tP, "launches": lP,
                                 "overhead_vs_single": tP / t1 - 1.0, "u_rel_diff_vs_single": d}
        del S, xs
        gc.collect()
        torch.cuda.empty_cache()
        print(c, w, res[f"emulated_x{w}"], file=sys.stderr, flush=True)
    out[f"cfg{c}"] = res
print(json.dumps(out))
