"""Pin the CPU oracle (oracle/mfwq_oracle.py) against the reference's own outputs.

The fixtures in tests/golden were produced by running igamf 0.1.0 itself
(tests/golden/make_golden.py).  CPU-only; no GPU needed.
"""
import numpy as np

from oracle import mfwq_oracle as O

SHEAR = [[1.0, 0.3, 0.1], [0.0, 1.2, 0.2], [0.0, 0.0, 0.9]]


def _oracle_problem(g):
    kv = O.Knots(int(g["p"]), g["knots"])
    rule = O.rule_1d(kv)
    rules = [rule] * 3
    C = O.stiffness_coeffs(rules, O.jac_for(g["geom"], SHEAR))
    return kv, rule, rules, O.Stiffness(rules, C)


def test_rule_factors_match_reference(golden):
    name, g = golden
    kv, rule, _, _ = _oracle_problem(g)
    assert np.array_equal(rule.pts, g["pts"])
    for ab in ((0, 0), (0, 1), (1, 0), (1, 1)):
        ref = g["W%d%d" % ab].toarray()
        got = rule.W[ab].toarray()
        assert got.shape == ref.shape
        assert np.abs(got - ref).max() <= 1e-13 * max(1.0, np.abs(ref).max()), (name, ab)
    for b in (0, 1):
        assert np.abs(rule.B[b].toarray() - g["B%d" % b].toarray()).max() <= 1e-14


def test_matvec_and_flops_match_reference(golden):
    name, g = golden
    _, _, rules, A = _oracle_problem(g)
    x = np.random.default_rng(0).standard_normal(A.N)
    fl = [0]
    y = A.apply(x, fl)
    ref = g["y"]
    assert np.linalg.norm(y - ref) <= 1e-13 * np.linalg.norm(ref), name
    assert fl[0] == int(g["flops"])
    assert O.matvec_flops_closed_form(rules) == int(g["flops"])


def test_fd_and_pcg_match_reference(golden):
    name, g = golden
    if "fd_y" not in g:
        return
    kv, _, _, A = _oracle_problem(g)
    P = O.FD([kv] * 3)
    x = np.random.default_rng(0).standard_normal(A.N)
    z = P.apply(x)
    assert np.linalg.norm(z - g["fd_y"]) <= 1e-12 * np.linalg.norm(g["fd_y"]), name
    if "u" in g:
        u, it, hist, conv, nmv, npc = O.pcg(A.apply, g["b"], P.apply, tol=1e-8)
        assert conv
        assert abs(it - int(g["iters"])) <= 1
        assert np.linalg.norm(u - g["u"]) <= 1e-9 * np.linalg.norm(g["u"])
        assert (nmv, npc) == (int(g["matvecs"]), int(g["precs"])) or abs(it - int(g["iters"])) == 1


def test_bicgstab_matches_reference():
    """Oracle BiCGStab (restating solvers.py:176-249) vs the reference's own runs, including the
    breakdown -> seeded restart -> failure path on a skew operator."""
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "solvers", "bicgstab_golden.npz"))
    from conftest import load_golden
    g = load_golden("ring_p3_n8")
    kv, _, _, A = _oracle_problem(g)
    P = O.FD([kv] * 3)
    b = np.random.default_rng(1).standard_normal(A.N)
    cases = {"ring_fd": (A.apply, b, P.apply, {}), "ring_nop_maxit5": (A.apply, b, None, {"maxit": 5}),
             "skew": (O.skew_blocks(64), z["skew_b"], None, {})}
    for tag, (op, rhs, pre, kw) in cases.items():
        x, it, hist, conv, nmv, npc = O.bicgstab(op, rhs, pre, tol=1e-8, **kw)
        meta = z[f"{tag}_meta"]
        assert [it, int(conv), nmv, npc] == meta.tolist(), tag
        ref_hist = z[f"{tag}_hist"]
        assert len(hist) == len(ref_hist)
        assert np.allclose(hist, ref_hist, rtol=1e-6, atol=1e-12), tag
        xr = z[f"{tag}_x"]
        assert np.linalg.norm(x - xr) <= 1e-9 * max(np.linalg.norm(xr), 1e-300), tag


def test_mass_and_system_match_reference():
    """Oracle mass operator / apply_system (operators.py:46-61, 87-132, 231-245) vs reference runs."""
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "solvers", "mass_golden.npz"))
    kv = O.uniform_knots(3, 8)
    rules = [O.rule_1d(kv)] * 3
    x = np.random.default_rng(0).standard_normal(O.Stiffness(rules, O.stiffness_coeffs(rules, O.jac_ring)).N)
    geo = {"ring": (O.jac_ring, O.map_ring), "shear": (O.jac_affine(SHEAR), O.map_affine(SHEAR))}
    alphas = {"const": 2.5, "field": lambda X: 1.0 + X[:, 0] ** 2 + 0.5 * X[:, 2]}
    for gname, (jac, fmap) in geo.items():
        K = O.Stiffness(rules, O.stiffness_coeffs(rules, jac))
        for aname, alpha in alphas.items():
            Mo = O.Mass(rules, O.mass_coeff(rules, jac, alpha, fmap))
            fl = [0]
            y = Mo.apply(x, fl)
            ref = z[f"{gname}_{aname}_y"]
            assert np.linalg.norm(y - ref) <= 1e-13 * np.linalg.norm(ref), (gname, aname)
            assert fl[0] == int(z[f"{gname}_{aname}_flops"])
            fl = [0]
            w = O.apply_system(Mo, K, x, alpha, fl)
            ref = z[f"{gname}_{aname}_sys"]
            assert np.linalg.norm(w - ref) <= 1e-13 * np.linalg.norm(ref), (gname, aname)
            assert fl[0] == int(z[f"{gname}_{aname}_sysflops"])
