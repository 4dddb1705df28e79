"""Import shim: the reference's package name `bri` bound to paper_1612_00001_b200 (tests only).

Everything the reference's tests import from `bri` (reference pkg/src/bri/__init__.py:11-69)
resolves to this repo's implementation; no reference code is imported.
"""

from paper_1612_00001_b200 import *  # noqa: F401,F403
from paper_1612_00001_b200 import __version__  # noqa: F401
import paper_1612_00001_b200 as _impl

for _name in dir(_impl):
    if not _name.startswith("__"):
        globals()[_name] = getattr(_impl, _name)
