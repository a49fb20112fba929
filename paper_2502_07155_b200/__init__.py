"""B200-native hot path of Algorithm 2 of arXiv 2502.07155 (NFFT-like procedure for
bandlimited functions): C-ABI library libbnfft.so (csrc/, include/bnfft.h) + ctypes binding.

    from paper_2502_07155_b200 import bnfft      # raises ImportError if the .so is not built
    plan = bnfft.Plan(d=1, M=1 << 20, sigma=2.0, m=8, window="sinh", prec="c64")
"""
__all__ = ["bnfft", "build"]
