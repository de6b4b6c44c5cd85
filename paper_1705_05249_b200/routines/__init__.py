"""The GEMM routine surface: gemm, gemm_batched, gemm_strided_batched and the
Netlib host-array layer."""

from .extras import gemm_batched, gemm_strided_batched
from .level3 import gemm
from .netlib import default_context, netlib_call

__all__ = ["gemm", "gemm_batched", "gemm_strided_batched", "default_context", "netlib_call"]
