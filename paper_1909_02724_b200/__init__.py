"""B200-native iFDK hot path (arXiv 1909.02724): FDK cone-beam reconstruction.

The compute lives in ``libifdk.so`` (hand-written sm_100a CUDA behind the C ABI
of ``include/ifdk.h``); ``ifdk`` is its thin ctypes binding and ``dist`` the
multi-GPU drivers (k-slab split with row-band exchange, projection split with
reduce-scatter) over ``torch.distributed``; ``iterative`` runs SART / SIRT from the
back-projector and its transpose, the matched forward projector.
"""
from .ifdk import (  # noqa: F401
    Geometry,
    IfdkError,
    ifdk_backproject,
    ifdk_backproject_alg2,
    ifdk_backproject_reduce,
    ifdk_backproject_alg4,
    ifdk_filter,
    ifdk_fill,
    ifdk_filter_scatter,
    ifdk_forward_project,
    ifdk_reconstruct,
    ifdk_reconstruct_host,
    ifdk_reconstruct_slab_host,
    ifdk_mlem_ratio,
    ifdk_mlem_update,
    ifdk_sart_ratio,
    ifdk_sart_update,
    last_launch_count,
    set_bp_variant,
)
from .iterative import SART, mlem, sart  # noqa: F401
