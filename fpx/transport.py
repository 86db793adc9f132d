"""`fpx.transport` -> paper_2501_12349_b200.transport (drop-in alias of the reference module name)."""
import sys as _sys

from paper_2501_12349_b200 import transport as _impl

_sys.modules[__name__] = _impl
