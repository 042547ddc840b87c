"""B200-native (sm_100a) batched querying of a DL4MT/Nematus cGRU translation model, as used by
arXiv 1605.04809 as a phrase-based decoder feature.  The work runs in libnmt.so (hand-written
CUDA: tcgen05/TMA GEMMs, fused online log-softmax, MUFU attention, device-side state cache);
this package is its C-ABI binding."""
from .nmt import (NMT_PREC_BF16, NMT_PREC_FP32CLASS, Context, Ensemble, Model, NmtError, lib,  # noqa: F401
                  test_gemm)
