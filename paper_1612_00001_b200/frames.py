"""Frames: index bookkeeping of the BRI recursion (reference engine.py:65-154).

A frame names an n x n sub-grid of 1-based block indices plus the quadrant
it occupies in its parent.  Splitting keeps the anchor (frame position
(2,2)) fixed: children drop the last row/column, and B/C/D exchange the
first and third index (§3.1 "forward procedure").  No arithmetic
happens here; the host scheduler (`dag.py`) turns frames into device work.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

from .errors import FrameTooSmallError

__all__ = ["Quadrant", "Frame", "BranchPath", "root_frame", "split_frame", "frame_at", "PLAN"]


class Quadrant(Enum):
    A = "A"
    B = "B"
    C = "C"
    D = "D"

    @property
    def mirror(self) -> "Quadrant":
        """A<->D, B<->C: the quadrant an internal node with this label eliminates."""
        return _MIRROR[self]


_MIRROR = {Quadrant.A: Quadrant.D, Quadrant.D: Quadrant.A,
           Quadrant.B: Quadrant.C, Quadrant.C: Quadrant.B}

BranchPath = tuple  # tuple[Quadrant, ...], root label first

# Eliminating quadrant q: result = r - l @ inv(pivot) @ rt, roles (pivot, rt, l, r)
# fixed by position (engine.py:149-154): the result sits opposite the pivot.
PLAN = {
    Quadrant.D: (Quadrant.D, Quadrant.C, Quadrant.B, Quadrant.A),
    Quadrant.C: (Quadrant.C, Quadrant.D, Quadrant.A, Quadrant.B),
    Quadrant.B: (Quadrant.B, Quadrant.A, Quadrant.D, Quadrant.C),
    Quadrant.A: (Quadrant.A, Quadrant.B, Quadrant.C, Quadrant.D),
}


@dataclass(frozen=True)
class Frame:
    rows: tuple
    cols: tuple
    label: Quadrant

    def __post_init__(self):
        if len(self.rows) != len(self.cols):
            raise FrameTooSmallError(
                f"frame must be square: {len(self.rows)} rows vs {len(self.cols)} cols")
        if len(self.rows) < 2:
            raise FrameTooSmallError(f"frame needs at least 2 block rows, got {len(self.rows)}")

    @property
    def n(self) -> int:
        return len(self.rows)

    @property
    def anchor(self) -> tuple:
        return (self.rows[1], self.cols[1])


def root_frame(k: int) -> Frame:
    idx = tuple(range(1, k + 1))
    return Frame(idx, idx, Quadrant.A)


def _exchanged(ix: tuple) -> tuple:
    # drop the last index and swap the first with the third: (i3, i2, i4, ..., i_n)
    return (ix[2], ix[1]) + ix[3:]


def split_frame(frame: Frame) -> tuple:
    """Children (A, B, C, D) of order n-1 (engine.py:119-132)."""
    if frame.n < 3:
        raise FrameTooSmallError(f"cannot split a frame of {frame.n} block rows")
    r, c = frame.rows, frame.cols
    rx, cx = _exchanged(r), _exchanged(c)
    return (Frame(r[:-1], c[:-1], Quadrant.A), Frame(r[:-1], cx, Quadrant.B),
            Frame(rx, c[:-1], Quadrant.C), Frame(rx, cx, Quadrant.D))


def frame_at(k: int, path) -> Frame:
    """Replay a branch path from the root; path[0] must be A (engine.py:135-143)."""
    if not path or path[0] is not Quadrant.A:
        raise FrameTooSmallError(f"branch path must start at the root label A, got {path}")
    frame = root_frame(k)
    for label in path[1:]:
        frame = split_frame(frame)["ABCD".index(label.name)]
    return frame
