"""B200-native guided extension alignment (AGAThA, arXiv 2403.06478 hot path).

The compute path is the sm_100a CUDA library ``libagatha.so`` behind the C ABI in
``include/agatha.h``; ``agatha`` is the thin ctypes binding (argument marshalling
only).  There is no CPU fallback: importing ``agatha`` without the built library, or
creating a context without an sm_100 GPU, raises.
"""
__all__ = ["agatha", "build"]
