"""B200-native Hydraulis two-stage data assignment (arxiv 2412.07894).

Product path: ``include/hyd.h`` C ABI -> ``libhyd.so`` (sm_100a kernels in ``csrc/``),
bound by ``hyd.py`` (marshalling only) and driven by ``assign.py``.  There is no CPU
fallback; the CPU oracle in ``oracle/`` is test infrastructure and is never imported here.
"""
from . import hyd  # noqa: F401

__all__ = ["hyd", "assign"]
