"""paper_2604_25936_b200 -- B200-native (sm_100a) engine for SAND's adaptive-depth T-MLP query path.

The product is libsand.so (csrc/, C ABI in include/sand.h); this package is a thin ctypes binding.
"""
from .sand import (SandContext, SandError, load_library, abi_version, EXPORTS,
                   SAND_FP32, SAND_BF16, SAND_TF32X3, SAND_F16X3, SAND_TAIL_LINEAR, SAND_TAIL_MULT,
                   SAND_DEPTH_NONFINITE, SAND_OPT_PAIR_KERNEL, SAND_OPT_DYN_SCHEDULE, SAND_OPT_KPROF, SAND_OPT_FP32_TENSOR)

__all__ = ["SandContext", "SandError", "load_library", "abi_version", "EXPORTS", "SAND_FP32", "SAND_BF16",
           "SAND_TF32X3", "SAND_F16X3", "SAND_TAIL_LINEAR", "SAND_TAIL_MULT", "SAND_DEPTH_NONFINITE",
           "SAND_OPT_PAIR_KERNEL", "SAND_OPT_DYN_SCHEDULE", "SAND_OPT_KPROF",
           "SAND_OPT_FP32_TENSOR"]
