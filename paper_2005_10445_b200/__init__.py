"""B200-native acquisition-mode ToA hot path of the ATLAS tag DSP
(arXiv 2005.10445; reference: /root/reference/proj "tagdsp").

The product is libtagdsp_gpu.so (hand-written sm_100a kernels behind the
C-ABI in include/tagdsp_gpu.h); capi.py mirrors the reference detector API
over it for Python callers and tests."""
from . import capi  # noqa: F401
from ._abi import DETECTION_DTYPE, demod_config, desk_config  # noqa: F401

__all__ = ["capi", "DETECTION_DTYPE", "demod_config", "desk_config"]
