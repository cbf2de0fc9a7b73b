"""B200-native sliCQ (arXiv 1210.0084): forward/inverse constant-Q NSGT applied slice by slice.

The product is ``libslicq.so`` (C ABI in ``include/slicq.h``: plan_create,
slicq_forward, slicq_inverse, plan_destroy, ...), hand-written sm_100a CUDA.
This package is its thin Python binding plus the multi-GPU slice-range driver.
"""
from ._lib import LIB_PATH, SlicqError, lib  # noqa: F401


def __getattr__(name):
    # torch-dependent parts load lazily so that `import paper_1210_0084_b200` stays cheap
    if name in ("Plan", "plan_for_config"):
        from . import api
        return getattr(api, name)
    raise AttributeError(name)
