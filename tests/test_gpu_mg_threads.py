"""pbit_sort_list_mg at G = 2..8 ranks on the one GPU available: the real mg.cu kernels and
host code, with an in-process stand-in for the NCCL transport (tests/fake_nccl), one host
thread per rank; every case is compared bit for bit with the oracle
(tests/fake_nccl/run_mg_threads.py).  Runs in a subprocess so that the test build of the
library (linked without NCCL) is the one loaded."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("transport", ["peer", "hybrid", "nccl"])
def test_mg_multi_rank_threads_vs_oracle(cuda_ok, transport):
    """Both transports (N4 peer windows, and the NCCL reference) bit-exact with the oracle,
    hence with each other."""
    env = dict(os.environ, PBIT_MG_TRANSPORT=transport)
    r = subprocess.run([sys.executable, os.path.join(HERE, "fake_nccl", "run_mg_threads.py")],
                       capture_output=True, text=True, timeout=900, env=env)
    print(r.stdout[-4000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "cases bit-exact" in r.stdout and "FAILED" not in r.stdout
    assert f"ok ({transport})" in r.stdout
