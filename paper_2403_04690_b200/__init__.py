"""B200-native fused neighborhood attention (arXiv 2403.04690).

The product is the C-ABI library ``libna.so`` (``include/na.h``), built
in-tree for sm_100a by ``paper_2403_04690_b200.build``.  This package is a
thin ctypes binding with the same names: it marshals torch CUDA tensors into
the ABI (pointers, sizes, the current CUDA stream) and does no arithmetic.
If the library is missing the import fails loudly; there is no CPU fallback.
"""
from .na import (NA_BF16, NA_F16, NA_F32, NA_IMPL_AUTO, NA_IMPL_SIMT, NA_IMPL_TC, NAError,
                 Problem, last_launch_count, lib, make_problem, na_bf16_precise, na_bwd,
                 na_bwd_workspace_size,
                 na_fwd, na_get_plan_choice, na_plan_candidates, na_selected_impl,
                 na_set_plan_choice, na_tune, na_validate, profile_collect, profile_enable,
                 status_string)

__all__ = ["NA_BF16", "NA_F16", "NA_F32", "NA_IMPL_AUTO", "NA_IMPL_SIMT", "NA_IMPL_TC", "NAError",
           "Problem", "last_launch_count", "lib", "make_problem", "na_bf16_precise", "na_bwd",
           "na_bwd_workspace_size", "na_fwd", "na_get_plan_choice", "na_plan_candidates",
           "na_selected_impl", "na_set_plan_choice", "na_tune", "na_validate", "profile_collect",
           "profile_enable", "status_string"]
