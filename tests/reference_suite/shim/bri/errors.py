"""Shim module: bri.errors -> paper_1612_00001_b200 (tests only)."""

import paper_1612_00001_b200 as _impl
from paper_1612_00001_b200 import errors as _mod

for _src in (_impl, _mod):
    for _name in dir(_src):
        if not _name.startswith("__"):
            globals()[_name] = getattr(_src, _name)
