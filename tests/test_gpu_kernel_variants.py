"""The fused matvec has two kernels (fused2.cu: phased, fused3.cu: warp-specialised) and a measured
dispatch between them.  The library reads MFWQ_F3 once per process, so each forced mode runs the
matvec parity files in its own interpreter: 0 = the phased kernel everywhere, 2 = the warp-specialised
kernel wherever it exists (p <= 6, three- and five-term sets, stored and on the fly, slabs)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FILES = ["tests/test_gpu_parity.py", "tests/test_gpu_otf.py", "tests/test_gpu_slab.py"]


@pytest.mark.parametrize("mode", ["0", "2"])
def test_parity_with_forced_kernel(mode):
    env = dict(os.environ, MFWQ_F3=mode)
    r = subprocess.run([sys.executable, "-m", "pytest", *FILES, "-x", "-q", "-m", "gpu", "-p", "no:cacheprovider"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
