"""Shim module: bri.engine -> paper_1612_00001_b200 (tests only)."""

import paper_1612_00001_b200 as _impl
from paper_1612_00001_b200 import engine as _mod
from paper_1612_00001_b200 import frames as _frames

for _src in (_impl, _mod) + ((_frames,) if "_frames" in globals() else ()):
    for _name in dir(_src):
        if not _name.startswith("__"):
            globals()[_name] = getattr(_src, _name)
