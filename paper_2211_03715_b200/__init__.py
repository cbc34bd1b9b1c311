"""B200-native (sm_100a) Tucker-format (TKD) convolution layer -- arXiv 2211.03715.

The compute path lives in ``libtdc.so`` (``csrc/``), exposed through the C-ABI
in ``include/tdc.h`` and bound by :mod:`paper_2211_03715_b200.tdc`.  Import
that module explicitly; it raises if the CUDA library is not built (there is
no CPU fallback).
"""
__all__ = ["tdc"]
