"""B200-native preprocessed-GENP / randomized low-rank hot path of arXiv
1406.5802 (reference: `randla`).

    include/randla_capi.h        C ABI (the drop-in boundary)
    include/randla_b200/*.hpp    C++ header API with the reference signatures
    paper_1406_5802_b200/csrc    sm_100a CUDA kernels + the ABI implementation
    paper_1406_5802_b200/randla  reference-shaped Python API over the ABI

Importing this package loads librandla_b200.so; it raises when the library
has not been built (there is no CPU fallback).
"""
from . import capi
from .randla import *  # noqa: F401,F403

capi.lib()
