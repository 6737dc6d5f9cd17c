"""Reads before first writes: the GPU parity cases re-run in a child process
whose device buffers are filled with +3.4e38 floats (and NaN) at allocation
(TDG_POISON_ALLOC, see DevBuf::ensure).  Any kernel that consumes memory it
(or an earlier stage) has not written -- e.g. an L2 discard that reaches into
a neighbouring tile -- turns into a wrong peak or a non-finite statistic and
fails the parity assertions."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("byte", ["0x7f", "0xff"])
def test_parity_with_poisoned_allocations(byte):
    if os.environ.get("TDG_POISON_ALLOC"):
        pytest.skip("already inside a poisoned run")
    env = dict(os.environ, TDG_POISON_ALLOC=byte)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(HERE, "test_gpu_parity.py"), os.path.join(HERE, "test_gpu_ring.py")],
                       env=env, capture_output=True, text=True, timeout=900)
    failed = [l for l in r.stdout.splitlines() if l.startswith(("FAILED", "ERROR", "E "))]
    assert r.returncode == 0, ("\n".join(failed[:40]), r.stderr[-2000:])
