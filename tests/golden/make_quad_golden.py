"""Golden fixtures for the load vector and error norms, produced by the REFERENCE (igamf 0.1.0):
``assemble_rhs`` (assembly.py:201-230), ``l2_relative_error`` / ``h1_relative_error`` and
``_error_integrals`` (problems.py:97-164) with the reference's sympy-derived cases.

    python tests/golden/make_quad_golden.py        # build container only (needs /root/reference)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from igamf import (TensorSpace, affine_map, assemble_rhs, build_tensor_rule, cg,  # noqa: E402
                   cube_sine_case, identity_map, make_uniform_knots, quarter_ring_map, setup_stiffness,
                   FDPreconditioner)
from igamf import problems as P  # noqa: E402

sys.path.insert(0, HERE)
from make_golden import SHEAR, perturbed  # noqa: E402

CASES = [
    # name, p, n_el, geometry, case, knots, gauss points per span for the rhs (None = p+1), solve?
    ("cube_p3_n4", 3, 4, "identity", "cube", None, None, True),
    ("ring_p2_n6", 2, 6, "ring", "osc", None, None, True),
    ("shear_p2_n3", 2, 3, "shear", "cube", None, 4, False),
    ("jitter_p3_n5", 3, 5, "identity", "cube", "jitter", None, False),
    ("ring_p6_n3", 6, 3, "ring", "osc", None, None, False),
]

for name, p, n_el, gk, ck, kk, gr, solve in CASES:
    kv = perturbed(p, n_el) if kk == "jitter" else make_uniform_knots(p, n_el)
    space = TensorSpace((kv,) * 3)
    geom = {"identity": identity_map(3), "ring": quarter_ring_map(),
            "shear": affine_map(np.array(SHEAR), np.array([0.2, -0.1, 0.3]))}[gk]
    case = cube_sine_case() if ck == "cube" else P.oscillating_case()
    rhs = assemble_rhs(space, geom, case.f, gauss_pts_per_span=gr)
    if solve:
        A = setup_stiffness(space, build_tensor_rule(space), geom)
        u, _ = cg(A.apply, rhs, FDPreconditioner(space).apply, tol=1e-10)
    else:
        u = np.random.default_rng(3).standard_normal(space.n_dofs) * 0.01
    g = p + 2
    e2l, r2l = P._error_integrals(space, geom, u, case, g, False)
    e2h, r2h = P._error_integrals(space, geom, u, case, g, True)
    np.savez_compressed(os.path.join(HERE, "quad", name + ".npz"), p=p, n_el=n_el, geom=gk, case=ck,
                        knots=np.asarray(kv.knots), rhs_gpts=-1 if gr is None else gr, rhs=rhs, u=u,
                        l2=P.l2_relative_error(space, geom, u, case), h1=P.h1_relative_error(space, geom, u, case),
                        err_l2=np.array([e2l, r2l]), err_h1=np.array([e2h, r2h]),
                        shear_b=np.array([0.2, -0.1, 0.3]))
    print(name, "rhs norm %.10e" % np.linalg.norm(rhs), "l2 %.3e h1 %.3e" % (np.sqrt(e2l / r2l), np.sqrt(e2h / r2h)))
