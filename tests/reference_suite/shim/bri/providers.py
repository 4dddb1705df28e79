"""Shim module: bri.providers -> paper_1612_00001_b200.providers (tests only).

`_run_maps` (reference providers.py:245-271, the padded-layout element maps) is
`window_maps` here."""

import paper_1612_00001_b200 as _impl
from paper_1612_00001_b200 import providers as _mod

for _src in (_impl, _mod):
    for _name in dir(_src):
        if not _name.startswith("__"):
            globals()[_name] = getattr(_src, _name)

_run_maps = _mod.window_maps
