"""B200-native (sm_100a) server-side HE convolution of SecONNds (arXiv 2506.11586).

The product is the C-ABI library ``libsecn.so`` (include/secn.h, sources in ``csrc/``);
``secn`` is its thin ctypes binding over torch CUDA tensors/streams and ``dist`` the
multi-GPU output-channel sharding with an NCCL all-gather of the server's output shares.
"""
from .secn import (DEFAULT_LOG_N, DEFAULT_PRIMES, DEFAULT_PRIMES32, DEFAULT_T_BITS, Context, FcPlan, MaskGen,
                   Plan, SecnError, conv_plan, fc_plan, lib)

__all__ = ["Context", "FcPlan", "MaskGen", "Plan", "SecnError", "conv_plan", "fc_plan", "lib", "DEFAULT_LOG_N",
           "DEFAULT_PRIMES", "DEFAULT_PRIMES32", "DEFAULT_T_BITS"]
