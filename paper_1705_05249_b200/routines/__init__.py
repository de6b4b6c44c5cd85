"""The GEMM routine surface: gemm, gemm_batched, gemm_strided_batched, the
Netlib host-array layer, and im2col (the convolution-lowering routine the C3
shapes come from)."""

from .extras import gemm_batched, gemm_strided_batched
from .im2col import convgemm, im2col
from .level3 import gemm
from .level3_structured import hemm, her2k, herk, symm, syr2k, syrk, trmm, trsm
from .netlib import default_context, netlib_call

__all__ = ["gemm", "gemm_batched", "gemm_strided_batched", "im2col", "convgemm", "default_context", "netlib_call",
           "symm", "hemm", "syrk", "herk", "syr2k", "her2k", "trmm", "trsm"]
