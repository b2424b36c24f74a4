"""ucores-b200: B200-native engine for SparkCL's mapCL / mapCLPartition /
reduceCL hot path (reference: the header-only C++20 `ucores` library).

  include/ucores_cuda.h          C-ABI of the CUDA library (the drop-in boundary)
  paper_1505_01120_b200/csrc     sm_100a kernels + runtime   -> _lib/libucores_cuda.so
  paper_1505_01120_b200/host     C++ seam adapters for the reference Engine
  capi / ops / pipeline          Python binding used by bench.py and the tests
"""
from .errors import (ArityMismatch, DeviceUnavailable, EmptyDataset, Error, JobFailed, KernelPanic,
                     LengthMismatch, UnknownKernel)

__all__ = ["ArityMismatch", "DeviceUnavailable", "EmptyDataset", "Error", "JobFailed", "KernelPanic",
           "LengthMismatch", "UnknownKernel"]
