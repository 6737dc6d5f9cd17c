import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run on the GPU box via gpurun)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def gpu_ctx():
    from paper_2005_10445_b200 import capi
    ctx = capi.Context(0)
    yield ctx
    import gc
    gc.collect()   # release code sets / windows before their context
    ctx.close()


@pytest.fixture(scope="session")
def ref():
    import refpy
    if not refpy.available():
        pytest.skip("oracle/_ref/libtagdsp_ref.so not built (make -C oracle ref)")
    return refpy
