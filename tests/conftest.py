import glob
import os
import sys

import numpy as np
import pytest
import scipy.sparse as sp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def golden_names():
    return sorted(os.path.basename(f)[:-4] for f in glob.glob(os.path.join(GOLDEN, "*.npz")))


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)
    d = {k: z[k] for k in z.files}
    for key in ("W00", "W01", "W10", "W11", "B0", "B1"):
        d[key] = sp.csr_matrix((d[key + "_data"], d[key + "_indices"], d[key + "_indptr"]),
                               shape=tuple(d[key + "_shape"]))
    d["geom"] = str(d["geom"])
    return d


@pytest.fixture(params=golden_names())
def golden(request):
    return request.param, load_golden(request.param)
