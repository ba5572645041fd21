"""B200-native disaggregated LBM solver path (arXiv 2503.07898).

Drop-in for the reference's dense / block-sparse / multi-resolution step
operators. All compute runs in the in-tree CUDA library
``_lib/libvoxl_b200.so`` behind the C-ABI ``include/voxl_b200.h``; importing
this package fails loudly when that library is missing.
"""
from ._capi import (LIB_PATH, VoxlCudaError, VoxlDomainError, VoxlError, VoxlInstability,  # noqa: F401
                    VoxlInvalidArgument, VoxlOutOfRange)
from .dense import (DenseEngine, classify_voxels, decompose, lattice_json, layout_addresses,  # noqa: F401
                    layout_json, make_desc, plan_ledger)
from .sparse import SparseEngine, SparsePlan, dispatch_plan_json, obstacle_mask  # noqa: F401
from .multires import MultiResEngine, MultiResPlan, band_level_map  # noqa: F401

__all__ = ["DenseEngine", "classify_voxels", "decompose", "lattice_json", "layout_addresses", "layout_json", "make_desc", "plan_ledger",
           "VoxlError", "VoxlInstability", "VoxlInvalidArgument", "VoxlOutOfRange", "VoxlCudaError",
           "VoxlDomainError", "LIB_PATH"]
