"""B200-native (sm_100a) hot path of distributed K-FAC (Osawa et al., arXiv 1811.12019).

The work lives in libkfac.so behind the C-ABI of include/kfac.h; this package is
its thin ctypes binding (``kfac``) and a step driver (``KfacStep``).  Importing
fails loudly when libkfac.so has not been built: there is no CPU fallback.
"""
from . import kfac  # noqa: F401  (raises ImportError when libkfac.so is missing)
from .kfac import (BF16, FP16, LPT, RR, Comm, KfacError, Plan, allgather_precond, comm_unique_id,  # noqa: F401
                   damped_inverse, factor_A, factor_all, factor_G, factor_ws_bytes, precondition,
                   reduce_scatter_factors, factor_diff, refresh, refresh_interval, RAMPUP, STEP13, update, bn_grads, bn_precondition, bn_ws_bytes, bn_exchange,
                   INV_AUTO, INV_FP64, INV_INT8, inverse_report, RS_PADDED, RS_PER_OWNER, WIRE_FP32, WIRE_FP16)
from .step import KfacStep  # noqa: F401
