"""CPU-only tests of the native host code and the C-ABI surface (no GPU needed).

* the C++ WQ rule builder (wq.py:62-164 replacement) against the reference's
  own factors in tests/golden (bit-exact collocation, conditioning-limited WQ
  weights),
* the native exact 1D stiffness/mass (solvers.py:48-62) against the oracle,
* every symbol declared in include/mfwq.h is exported by libmfwq.so,
* error mapping onto the reference's exception types.
"""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1712_08565_b200 as M
from paper_1712_08565_b200 import _lib
from paper_1712_08565_b200.splines import KnotVector
from oracle import mfwq_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# relative tolerance of the built-in Jacobi-SVD row solver (used only when no host LAPACK is
# registered): the per-row least-squares systems lose accuracy like 1/sigma_min (the smallest kept
# singular value is 0.23, 1.7e-3, 1.5e-6, 3e-10, 1.8e-14 of the largest for p = 2, 4, 6, 8, 10)
JACOBI_W_TOL = {1: 1e-13, 2: 1e-13, 3: 1e-13, 4: 1e-13, 5: 1e-12, 6: 1e-9, 8: 1e-7}


def test_rule_builder_matches_reference(golden):
    """With numpy's LAPACK registered (the default), the native builder solves every row with the
    reference's own driver and calling sequence (np.linalg.lstsq -> dgelsd, wq.py:97) on
    bit-identical right-hand sides (numpy's leggauss -> exact Gram, wq.py:41-59): the points,
    collocation and WQ weights equal the reference's bit for bit, at every degree incl. p = 8, 10."""
    name, g = golden
    p = int(g["p"])
    assert _lib.lib().mfwq_lapack_active() == 1
    r = M.build_wq_rule(KnotVector(p, g["knots"]))
    assert np.array_equal(r.points, g["pts"])
    for b in (0, 1):  # Cox-de Boor collocation
        A, B = r.colloc[b], g["B%d" % b]
        assert np.array_equal(A.indptr, B.indptr) and np.array_equal(A.indices, B.indices)
        assert np.array_equal(A.data, B.data), (name, b)
    for ab in ((0, 0), (0, 1), (1, 0), (1, 1)):
        A, B = r.weights[ab], g["W%d%d" % ab]
        assert np.array_equal(A.indptr, B.indptr) and np.array_equal(A.indices, B.indices)
        assert np.array_equal(A.data, B.data), (name, ab, np.abs(A.data - B.data).max())


def test_rule_builder_jacobi_path_within_conditioning():
    """The self-contained row solver (no host LAPACK: a C-ABI consumer without numpy) agrees with
    the reference's weights to the conditioning of the row systems."""
    import subprocess
    import sys
    code = (
        "import sys, numpy as np; sys.path[:0] = [%r, %r]\n"
        "import paper_1712_08565_b200 as M\nfrom paper_1712_08565_b200 import _lib\n"
        "from conftest import load_golden, golden_names\n"
        "assert _lib.lib().mfwq_lapack_active() == 0\n"
        "tol = %r\n"
        "for name in golden_names():\n"
        "    g = load_golden(name); p = int(g['p'])\n"
        "    if p not in tol: continue\n"
        "    r = M.build_wq_rule(M.KnotVector(p, g['knots']))\n"
        "    for ab in ((0, 0), (0, 1), (1, 0), (1, 1)):\n"
        "        A, B = r.weights[ab].toarray(), g['W%%d%%d' %% ab].toarray()\n"
        "        err = np.abs(A - B).max() / np.abs(B).max()\n"
        "        assert err <= tol[p], (name, ab, err)\n"
        "print('ok')\n") % (ROOT, os.path.join(ROOT, "tests"), JACOBI_W_TOL)
    env = dict(os.environ, MFWQ_NO_NUMPY_LAPACK="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


@pytest.mark.parametrize("p,n_el", [(1, 3), (2, 5), (3, 7), (4, 9), (6, 6), (10, 10)])
def test_rule_exactness(p, n_el):
    """Every row satisfies its exactness system (wq.py:115-116), checked with the oracle's Gram."""
    kv = O.uniform_knots(p, n_el)
    r = M.build_wq_rule(KnotVector(p, kv.t))
    for (a, b), W in r.weights.items():
        G = O.gram(kv, a, b)
        Cb = O.collocation(kv, r.points, b).toarray()  # (npts, nfun)
        lhs = W.toarray() @ Cb                          # sum_q W[i,q] D^b b_j(x_q)
        for i in range(kv.nfun):
            lo, hi = kv.supp(i)
            js = [j for j in range(kv.nfun) if kv.supp(j)[1] > lo + 1e-14 and kv.supp(j)[0] < hi - 1e-14]
            assert np.abs(lhs[i, js] - G[i, js]).max() <= 1e-10


@pytest.mark.parametrize("p,n_el", [(1, 4), (3, 8), (4, 8), (8, 12)])
def test_univariate_km_matches_oracle(p, n_el):
    kv = M.make_uniform_knots(p, n_el)
    K, Mm = M.univariate_parametric_matrices(kv)
    Ko, Mo = O.univariate_KM(O.uniform_knots(p, n_el))
    assert np.abs(K - Ko).max() <= 1e-12 * np.abs(Ko).max()
    assert np.abs(Mm - Mo).max() <= 1e-14 * np.abs(Mo).max()


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "mfwq.h")).read()
    declared = set(re.findall(r"\b(mfwq_[a-z0-9_]+)\s*\(", hdr))
    so = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in sorted(declared) if not hasattr(so, s)]
    assert not missing, missing
    assert declared <= set(_lib.EXPORTED) | {"mfwq_version"}


def test_error_mapping():
    with pytest.raises(ValueError):  # not open
        M.build_wq_rule(type("KV", (), {"degree": 2, "knots": np.array([0, 0.5, 0.5, 1.0, 1, 1])})())
    bad = np.array([0, 0, 0, 0.5, 0.5, 1, 1, 1.0])  # interior multiplicity 2
    with pytest.raises(ValueError):
        M.build_wq_rule(type("KV", (), {"degree": 2, "knots": bad})())
    with pytest.raises(ValueError):
        M.make_uniform_knots(0, 4)
    assert _lib.lib().mfwq_version() == 1


def test_space_and_index_maps():
    sp = M.tensor_space(3, 4, 3)
    assert sp.n_per_dir == (5, 5, 5) and sp.n_dofs == 125
    assert M.multi_to_scalar((2, 1, 1), (5, 5, 5)) == 2
    assert M.scalar_to_multi(M.multi_to_scalar((3, 4, 5), (5, 5, 5)), (5, 5, 5)) == (3, 4, 5)


def test_bench_reference_arm_runs_on_host_cores():
    """bench.py --impl reference: the CPU arm (oracle matvec processes on the host cores) prints one
    JSON line in the driver's format, with its own e2e and cpu_baseline."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MFWQ_REF_WORKERS="2")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1"], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "DoF/s" and line["value"] > 0
    assert line["cpu_baseline"]["cores"] == 2 and line["cpu_baseline"]["kind"] == "port"
    assert line["e2e"]["value"] == line["value"] and line["e2e"]["h2d_bytes_per_step"] == 0
    assert set(line["per_degree_s"]) == {"2", "3"}


def test_bench_reference_arm_slab_headline_under_torchrun():
    """bench.py --impl reference at N = 2 (launched like the driver does, through torchrun): rank 0
    times the oracle's PCG iteration on a z-slab sample of the cfg5 problem and prints one line with the
    N > 1 headline's metric; rank 1 exits 0 without work."""
    import json
    import socket
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ, MFWQ_SLAB_SAMPLE_NXY="6", MFWQ_SLAB_SAMPLE_EL="2")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(root, "bench.py"),
                        "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["scaling"] == "strong" and line["value"] > 0
    assert line["metric"].startswith("MF-WQ cfg5 slab FD-PCG") and line["e2e"]["value"] == line["value"]
