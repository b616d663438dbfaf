"""B200-native (sm_100a) In-Place Activated BatchNorm hot path (arXiv 1712.02616).

The compute path is libiabn.so (hand-written CUDA: channel-resident cluster
kernels with TMA bulk copies and DSMEM reductions, plus a streaming schedule),
behind the C ABI of include/iabn.h.  This package is its thin Python binding.
"""
from . import _lib
from .functional import (Comm, InPlaceABN, InPlaceABNFunction, backward, backward_apply,
                         backward_reduce, backward_sync_emulated, fold_conv, forward,
                         forward_apply, forward_reduce, forward_sync_emulated, inplace_abn,
                         layout_of)

__all__ = ["Comm", "InPlaceABN", "InPlaceABNFunction", "backward", "backward_apply",
           "backward_reduce", "backward_sync_emulated", "fold_conv", "forward", "forward_apply",
           "forward_reduce", "forward_sync_emulated", "inplace_abn",
           "layout_of", "_lib"]
