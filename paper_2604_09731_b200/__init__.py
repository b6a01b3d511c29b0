"""B200-native SMART hot path (arXiv 2604.09731): C-ABI libsmart.so + thin binding.

    from paper_2604_09731_b200 import smart
    ctx = smart.Smart(smart.Config(...), smart.Cost(...))
"""
__all__ = ["smart"]
