"""fa3b: B200-native (sm_100a) FlashAttention-3 hot path.

The product is the CUDA library ``libfa3b.so`` behind the C ABI in
``include/fa3b.h``; ``api`` binds it for torch device tensors and
``flashlab`` mirrors the reference library's host API on top of it.
"""
__all__ = ["api", "build"]
