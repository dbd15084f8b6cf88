"""B200-native mixed-mode broadcast differentiation (arXiv 1810.08297).

The product is native: ``libbcad_cu.so`` (sm_100a kernels + the C-ABI of
``include/bcad_cu.h``) and the C++ drop-in host API in ``include/bcad/``.
This Python package only binds the C-ABI (``native``) and shards batches
across ranks (``partition``) for tests and ``bench.py``.
"""

__all__ = ["native"]
