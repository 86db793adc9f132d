"""`fpx.spatial_hash` -> paper_2501_12349_b200.spatial_hash (drop-in alias of the reference module name)."""
import sys as _sys

from paper_2501_12349_b200 import spatial_hash as _impl

_sys.modules[__name__] = _impl
