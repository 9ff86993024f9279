"""B200-native FGC entropic Gromov-Wasserstein hot path (arXiv 2404.08970).

The compute lives in ``libgwdp.so`` (hand-written sm_100a CUDA behind the C ABI in
``include/gwdp.h``); this package is the thin Python binding.  Importing it does not
touch the GPU; the first call loads the library and fails loudly if it is missing.
"""

from . import _lib  # noqa: F401

__all__ = ["grad", "sinkhorn", "solve", "solve_host", "ugw_solve", "Context", "Result", "plan_buffer",
           "GwError"]

GwError = _lib.GwError


def __getattr__(name):
    if name in ("grad", "sinkhorn", "solve", "solve_host", "ugw_solve", "Context", "Result", "plan_buffer"):
        from . import api
        return getattr(api, name)
    raise AttributeError(name)
