"""Measure the SURVEY §8(d) solver configurations beyond the bench's cfg 2/3 on one GPU.

    python tools/run_configs.py --cfg 4      # k-method sweep: (p, n_el) = (2,128) .. (10,120), N = 128^3
    python tools/run_configs.py --cfg 5      # p=6, n_el=512 quarter ring (137 M DoFs) on a single B200

Each case times the setup phases (WQ rule, coefficient grids, FD eigendecomposition) and the FD-PCG
solve to 1e-8 on b ~ N(0,1) seed 1, and compares ||u|| / iterations with the reference-oracle anchors
recorded in SURVEY §8(c) (cfg 4).  Prints one JSON object.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1712_08565_b200 as M  # noqa: E402

# oracle anchors (reference run): ||u||_2 and PCG iterations at cfg 4
CFG4 = {2: (128, 3.0208112873e+05, 27), 4: (126, 1.8017689318e+07, 27), 6: (124, 2.4482677025e+09, 28),
        8: (122, 4.5817363209e+11, 31), 10: (120, 1.0585471769e+14, 33)}

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, choices=[4, 5], required=True)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
dev = torch.device("cuda:0")
out = {"cfg": a.cfg, "gpu": torch.cuda.get_device_name(0), "cases": [],
       "note": "one small untimed case first, so CUDA context, module load and cuSOLVER initialisation "
               "are not charged to the first timed case's setup phases"}
bench.solve_case(M, torch, dev, 2, 8, reps=1)  # warm-up
if a.cfg == 4:
    for p, (n_el, unorm, iters) in CFG4.items():
        r = bench.solve_case(M, torch, dev, p, n_el, reps=a.reps)
        r["oracle"] = {"u_norm": unorm, "iterations": iters,
                       "u_norm_rel_diff": abs(r["u_norm"] - unorm) / unorm, "iter_diff": r["iterations"] - iters}
        out["cases"].append(r)
        print(json.dumps(r), file=sys.stderr, flush=True)
else:
    r = bench.solve_case(M, torch, dev, 6, 512, reps=1)
    out["cases"].append(r)
print(json.dumps(out))
