"""paper_2506_08781_b200 — B200-native batch verifier for POSLO (arXiv 2506.08781).

Drop-in for the reference's batch-verification path (agg_ekeys / paver,
/root/reference/proj/src/batch_verify.cpp) as hand-written sm_100a kernels
behind a C-ABI (include/poslo_gpu.h). `api` mirrors the reference interface.
"""
from .api import (  # noqa: F401
    DeviceError, EpochSignature, FormatError, PackedBatch, PoslocPublicKey, SeedNotDisclosed,
    SeedNode, SeedStack, StateError, SuiteConfig, Verifier, agg_ekeys, default_verifier, paver,
)

__version__ = "0.1.0"
