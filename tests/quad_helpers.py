"""Shared loaders for the load-vector / error-norm fixtures (tests/golden/quad, made by the reference)."""
import glob
import os

import numpy as np

from oracle import mfwq_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
QUAD = os.path.join(HERE, "golden", "quad")
SHEAR = [[1.0, 0.3, 0.1], [0.0, 1.2, 0.2], [0.0, 0.0, 0.9]]


def quad_names():
    return sorted(os.path.basename(f)[:-4] for f in glob.glob(os.path.join(QUAD, "*.npz")))


def load_quad(name):
    z = np.load(os.path.join(QUAD, name + ".npz"), allow_pickle=False)
    d = {k: z[k] for k in z.files}
    for k in ("geom", "case"):
        d[k] = str(d[k])
    d["rhs_gpts"] = int(d["rhs_gpts"])
    d["p"] = int(d["p"])
    return d


def oracle_geometry(g):
    """(map, jacobian) of the fixture's geometry, oracle side."""
    if g["geom"] == "identity":
        return (lambda xi: xi.copy()), O.jac_identity
    if g["geom"] == "ring":
        return O.map_ring, O.jac_ring
    A, b = np.array(SHEAR), np.asarray(g["shear_b"])
    return (lambda xi: xi @ A.T + b), O.jac_affine(A)


def oracle_case(g):
    return O.cube_sine() if g["case"] == "cube" else O.ring_oscillating()
