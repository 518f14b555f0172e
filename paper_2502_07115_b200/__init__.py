"""paper_2502_07115_b200 -- B200 (sm_100a) batched simulator of the online KV-cache-constrained
batch scheduler of arXiv 2502.07115 (MC-SF, Algorithm 1) and its baselines.

The product is libkvsched.so (C ABI in include/kvsched.h, CUDA kernels in csrc/); this
package holds its ctypes binding (kvsched.py), the nvcc build (build.py) and the multi-GPU
sharding helpers (dist.py).
"""
import os as _os

# The streamed host path runs a persistent kernel that polls per-chunk flags written by a copy
# stream's memory operations; give every stream its own hardware queue so a flag write is
# never queued behind that kernel (read when the CUDA context is created, so this only takes
# effect if nothing has initialised CUDA yet; a wait that gives up falls back to the chunked
# pipeline, see kvsched.cu).
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from .kvsched import (ALPHA, ALPHA_BETA, MC_BENCH, MCSF, Context, Policy, alloc_outputs, hints_of,
                      load, simulate, to_device)

__all__ = ["Context", "Policy", "load", "simulate", "alloc_outputs", "to_device", "hints_of",
           "MCSF", "MC_BENCH", "ALPHA", "ALPHA_BETA"]
