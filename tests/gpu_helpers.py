"""Helpers shared by the GPU parity tests."""
from types import SimpleNamespace

import numpy as np

import paper_1712_08565_b200 as M
from oracle import mfwq_oracle as O

SHEAR = [[1.0, 0.3, 0.1], [0.0, 1.2, 0.2], [0.0, 0.0, 0.9]]


def golden_rule(g):
    """A TensorRule-shaped object holding the REFERENCE's own 1D factors."""
    kv = M.KnotVector(int(g["p"]), g["knots"])
    r1 = SimpleNamespace(kv=kv, points=g["pts"], n_points=len(g["pts"]),
                         weights={ab: g["W%d%d" % ab] for ab in ((0, 0), (0, 1), (1, 0), (1, 1))},
                         colloc={0: g["B0"], 1: g["B1"]})
    return M.TensorRule((r1, r1, r1)), M.TensorSpace((kv, kv, kv))


def geom_of(kind):
    return {"identity": M.identity_map(3), "ring": M.quarter_ring_map(),
            "shear": M.affine_map(np.array(SHEAR), np.zeros(3))}[kind]


def relerr(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)
