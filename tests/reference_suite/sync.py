"""Copy the reference's own test suite next to the import shim (test infrastructure).

The reference tests (`/root/reference/pkg/tests/*.py`, 199 cases) are the drop-in proof
SURVEY.md §4/§7 asks for: they run unmodified against this package through `shim/bri`,
which binds the reference's import name `bri` to `paper_1612_00001_b200`.  The copy goes to
`vendored/` (git-ignored: it is the reference's source, not ours, and stays out of history;
it is not gpurun-ignored, so it travels to the GPU box with the snapshot).  `build()` in
`__graft_entry__.py` calls `sync()` whenever /root/reference is present.
"""

from __future__ import annotations

import os
import shutil

HERE = os.path.dirname(os.path.abspath(__file__))
REF_TESTS = "/root/reference/pkg/tests"
DEST = os.path.join(HERE, "vendored")


def sync(src: str = REF_TESTS, dest: str = DEST) -> int:
    if not os.path.isdir(src):
        return 0
    os.makedirs(dest, exist_ok=True)
    n = 0
    for name in sorted(os.listdir(src)):
        if name.endswith(".py"):
            shutil.copyfile(os.path.join(src, name), os.path.join(dest, name))
            n += 1
    with open(os.path.join(dest, "pytest.ini"), "w") as fh:
        fh.write("[pytest]\naddopts = -p no:cacheprovider\n")
    return n


if __name__ == "__main__":
    print(f"copied {sync()} files to {DEST}")
