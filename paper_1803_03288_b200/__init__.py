"""B200-native TicTac scheduling core (arXiv 1803.03288).

The product is `libcommsched.so` (include/commsched.h): the reference's C
interface with every scheduling and simulation computation on sm_100a
kernels. This package only binds it (capi.py). Importing raises when the
library has not been built — there is no Python or CPU fallback.
"""
from .capi import (CS_ERR_COVERAGE, CS_ERR_INTERNAL, CS_ERR_IO, CS_ERR_PARAMETER,  # noqa: F401
                   CS_ERR_VALIDATION, CS_OK, PRODUCT_LIB, CsError, Graph, Lib, Oracle, Report,
                   Schedule, SimPolicy, SweepPlan, SweepStats, policy)

_default = None


def lib() -> Lib:
    """The B200 library (loaded once)."""
    global _default
    if _default is None:
        _default = Lib(PRODUCT_LIB)
    return _default
