"""Pin the oracle's load vector and error integrals (oracle/mfwq_oracle.py) against the reference's
own outputs (tests/golden/quad, tests/golden/make_quad_golden.py).  CPU only."""
import numpy as np
import pytest

from oracle import mfwq_oracle as O
from quad_helpers import load_quad, oracle_case, oracle_geometry, quad_names


@pytest.mark.parametrize("name", quad_names())
def test_oracle_rhs_matches_reference(name):
    g = load_quad(name)
    kv = O.Knots(g["p"], g["knots"])
    fmap, jac = oracle_geometry(g)
    _, _, f = oracle_case(g)
    rhs = O.assemble_rhs([kv] * 3, fmap, jac, f, None if g["rhs_gpts"] < 0 else g["rhs_gpts"])
    assert np.linalg.norm(rhs - g["rhs"]) <= 1e-12 * np.linalg.norm(g["rhs"]), name


@pytest.mark.parametrize("name", quad_names())
@pytest.mark.parametrize("with_grad", [False, True])
def test_oracle_error_integrals_match_reference(name, with_grad):
    g = load_quad(name)
    kv = O.Knots(g["p"], g["knots"])
    fmap, jac = oracle_geometry(g)
    u, grad, _ = oracle_case(g)
    e2, r2 = O.error_integrals([kv] * 3, fmap, jac, g["u"], u, grad, g["p"] + 2, with_grad)
    ref = g["err_h1" if with_grad else "err_l2"]
    assert abs(e2 - ref[0]) <= 1e-12 * ref[0] and abs(r2 - ref[1]) <= 1e-12 * ref[1], (name, e2, r2, ref)
