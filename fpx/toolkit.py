"""`fpx.toolkit` -> paper_2501_12349_b200.toolkit (drop-in alias of the reference module name)."""
import sys as _sys

from paper_2501_12349_b200 import toolkit as _impl

_sys.modules[__name__] = _impl
