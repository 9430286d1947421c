"""B200-native (sm_100a) sparse speculative verification over Native Sparse
Attention: the hot path of arXiv 2605.19893 behind a C-ABI drop-in boundary
(include/specsv_b200/nsa_verify.h).  See DESIGN.md."""
from . import abi  # noqa: F401

__version__ = "0.1.0"


def build(force: bool = False) -> str:
    from .build import build as _b
    return _b(force=force)
