"""Full-size VECTOR anchors, produced by running the REFERENCE itself (igamf 0.1.0).

Run in the build container (the reference is absent on the GPU box); takes ~1 h and
~47 GB of RAM at cfg 3 (the reference's own coefficient setup, operators.py:64-84):

    python tests/golden/make_anchors.py [cfg2] [cfg4] [cfg3]

Each anchored vector v (a matvec output of ``StiffnessOperator.apply``, operators.py:185-204,
an FD apply, solvers.py:107-115, or a ``cg`` solution, solvers.py:137-173) is summarised by
size-independent fingerprints that pin the whole vector, not only its norm:

* ``norm``: ||v||_2 (17 significant digits),
* ``planes``: the 2-norm of every xi3 plane (n3 values: v viewed as (n3, n2, n1), kron.py:81-82),
* ``dots``: <v, r_k> for the 8 probe vectors r_k = default_rng(PROBE_SEED0 + k).standard_normal(N).

A vector u agrees with the anchor to relative tolerance t when every fingerprint does, measured
against ||v|| (planes: max_i |p_i - P_i| <= t ||v||; dots: |d_k - D_k| <= t ||v|| ||r_k||).
Inputs are the SURVEY §8(d) ones: x = default_rng(0), b = default_rng(1), N(0,1) fp64.
"""

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "full_vectors.json")
PROBE_SEED0 = 100
NPROBE = 8


def fingerprint(v, n3):
    v = np.asarray(v, dtype=float)
    N = v.size
    d = {"N": int(N), "norm": float(np.linalg.norm(v)),
         "planes": np.linalg.norm(v.reshape(n3, -1), axis=1).tolist(), "dots": [], "probe_norms": []}
    for k in range(NPROBE):
        r = np.random.default_rng(PROBE_SEED0 + k).standard_normal(N)
        d["dots"].append(float(r @ v))
        d["probe_norms"].append(float(np.linalg.norm(r)))
    return d


def _save(res):
    with open(OUT + ".tmp", "w") as fh:
        json.dump(res, fh, indent=0)
    os.replace(OUT + ".tmp", OUT)


def main(which):
    sys.path.insert(0, "/root/reference/pkg/src")
    import igamf
    from igamf import (FDPreconditioner, build_tensor_rule, cg, identity_map, quarter_ring_map,
                       setup_stiffness, tensor_space)
    print("reference igamf", igamf.__version__, "numpy", np.__version__, flush=True)
    res = json.load(open(OUT)) if os.path.exists(OUT) else {}

    def case(tag, p, n_el, geom, pcg, fd=False):
        t0 = time.time()
        space = tensor_space(p, n_el, 3)
        n3 = space.n_per_dir[2]
        A = setup_stiffness(space, build_tensor_rule(space), geom)
        x = np.random.default_rng(0).standard_normal(space.n_dofs)
        res[f"{tag}_Ax"] = fingerprint(A.apply(x), n3)
        print(tag, "Ax", res[f"{tag}_Ax"]["norm"], f"{time.time() - t0:.0f}s", flush=True)
        _save(res)
        if fd or pcg:
            P = FDPreconditioner(space)
        if fd:
            res[f"{tag}_fd"] = fingerprint(P.apply(x), n3)
            _save(res)
        if pcg:
            b = np.random.default_rng(1).standard_normal(space.n_dofs)
            u, rep = cg(A.apply, b, P.apply, tol=1e-8)
            d = fingerprint(u, n3)
            d.update(iterations=rep.iterations, converged=bool(rep.converged), final_res=rep.residuals[-1],
                     secs=time.time() - t0)
            res[f"{tag}_u"] = d
            print(tag, "u", d["norm"], rep.iterations, f"{time.time() - t0:.0f}s", flush=True)
            _save(res)

    if "cfg2" in which:
        for p in (2, 3, 4, 5, 6):
            case(f"cfg2_p{p}", p, 128, identity_map(3), pcg=False, fd=(p == 4))
    if "cfg4" in which:
        for p, n_el in ((2, 128), (4, 126), (6, 124), (8, 122), (10, 120)):
            case(f"cfg4_p{p}", p, n_el, quarter_ring_map(), pcg=True)
    if "cfg3" in which:
        case("cfg3", 4, 256, quarter_ring_map(), pcg=True, fd=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg2", "cfg4", "cfg3"])
