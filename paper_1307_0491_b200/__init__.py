"""B200-native time-stepping path for the coupled shallow-water + Exner
(Grass bedload) relaxation solver of arXiv 1307.0491.

The compute path is the CUDA library ``lib/libsilt_b200.so`` behind the C ABI
``include/silt_cuda.h``; this package only binds it (``native``), mirrors its
structures (``abi``), builds inputs (``scenarios``) and drives multi-GPU row
strips over torch.distributed (``distributed``).
"""
from . import abi  # noqa: F401

__all__ = ["abi"]
