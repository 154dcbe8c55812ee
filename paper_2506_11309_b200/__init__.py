"""B200-native (sm_100a) tree-verification step of SwiftSpec (arXiv 2506.11309).

The product is the C-ABI library libswiftspec.so (include/swiftspec.h) built
from csrc/ by `python -m paper_2506_11309_b200.build`; `swiftspec.py` is the
thin ctypes binding.  No CPU fallback exists.
"""
from .swiftspec import Shard, SwiftSpecError, lib, LIB_PATH, EXPORTS  # noqa: F401
