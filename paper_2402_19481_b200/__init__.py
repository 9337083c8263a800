"""B200-native displaced patch parallelism (DistriFusion, arXiv 2402.19481).

A drop-in for the reference's hot path (patchsim PatchRunner / run_sampling and
its per-layer operators): a C++ host runtime plus hand-written sm_100a kernels
behind the C ABI in ``include/pp_b200.h``.  This package is the Python mirror
of that interface (``patchsim`` names, argument meaning and error behaviour).
"""
from ._native import (CudaError, InvalidArgument, NcclError, PPError, RuntimeFailure,  # noqa: F401
                      lib)
