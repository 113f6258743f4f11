"""paper_2112_03804_b200 — B200-native gradient oracle for Kronecker-factored
river endgames (arXiv 2112.03804), a drop-in for the reference kronriver
library's GradientEngine boundary (solver.hpp:21-27) and solver step.

Native code:
  lib/libkrcuda.so  sm_100a kernels behind the kr_* C ABI (include/kr_engine.h)
  lib/libkrhost.so  C++ host side: instances, payoff, sparsifier, bundles
"""
from ._native import (ContractError, DegenerateBeliefsError, GuardError, InvalidInputError, KrError,
                      NoDeviceError, ParseError, device_count)
from .engine import CudaEngine

__all__ = ["CudaEngine", "KrError", "InvalidInputError", "ContractError", "GuardError", "ParseError",
           "DegenerateBeliefsError", "NoDeviceError", "device_count"]
