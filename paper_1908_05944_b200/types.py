"""Value types of the drop-in boundary (host side, no device work).

Mirrors the reference's public dataclasses so callers can switch imports:
``Ball`` / ``SimplexKey`` / ``TolerancePolicy`` / ``OrthoResult``
(reference: geometry.py:22-111) and ``simplex_compare`` (geometry.py:100-103).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Iterator


@dataclass(frozen=True)
class TolerancePolicy:
    """eps_abs: slack on every power-distance comparison (A^2, ties count as
    satisfied).  eps_singular: |pivot| at or below this flags an affinely
    dependent simplex.  Both must be > 0 (reference geometry.py:32-37)."""

    eps_abs: float = 1e-9
    eps_singular: float = 1e-12

    def __post_init__(self):
        if not (self.eps_abs > 0.0 and self.eps_singular > 0.0):
            raise ValueError("tolerances must be strictly positive")


DEFAULT_TOLERANCE = TolerancePolicy()


@dataclass(frozen=True)
class Ball:
    """Weighted point: centre (A), radius (A) and its input ordinal
    (reference geometry.py:43-63: finite centre, finite radius >= 0, index >= 0)."""

    center: tuple
    radius: float
    index: int = 0

    def __post_init__(self):
        xyz = tuple(float(v) for v in self.center)
        if len(xyz) != 3:
            raise ValueError("center must have exactly 3 components")
        if not (math.isfinite(xyz[0]) and math.isfinite(xyz[1]) and math.isfinite(xyz[2])):
            raise ValueError(f"ball {self.index}: non-finite center {xyz}")
        rad = float(self.radius)
        if not math.isfinite(rad) or rad < 0.0:
            raise ValueError(f"ball {self.index}: radius must be finite and >= 0")
        if self.index < 0:
            raise ValueError("index must be non-negative")
        object.__setattr__(self, "center", xyz)
        object.__setattr__(self, "radius", rad)


@dataclass(frozen=True)
class SimplexKey:
    """1..4 strictly increasing ball indices (reference geometry.py:66-97)."""

    vertices: tuple

    def __post_init__(self):
        vs = tuple(int(v) for v in self.vertices)
        if not 1 <= len(vs) <= 4:
            raise ValueError("a simplex has 1 to 4 vertices")
        if min(vs) < 0:
            raise ValueError("vertex indices must be non-negative")
        for lo, hi in zip(vs, vs[1:]):
            if lo >= hi:
                raise ValueError(f"vertices must be strictly increasing, got {vs}")
        object.__setattr__(self, "vertices", vs)

    @classmethod
    def of(cls, *indices: int) -> "SimplexKey":
        return cls(tuple(sorted(int(i) for i in indices)))

    @property
    def dim(self) -> int:
        return len(self.vertices) - 1

    def sort_key(self):
        return (self.dim, self.vertices)

    def facets(self) -> Iterator["SimplexKey"]:
        if self.dim > 0:
            for skip in range(len(self.vertices)):
                yield SimplexKey(tuple(v for i, v in enumerate(self.vertices) if i != skip))


def simplex_compare(a: SimplexKey, b: SimplexKey) -> int:
    """-1/0/+1 under (dimension, lexicographic vertices)."""
    ka, kb = a.sort_key(), b.sort_key()
    return (ka > kb) - (ka < kb)


@dataclass(frozen=True)
class OrthoResult:
    """Equal-power point and its power distance (A^2)."""

    center: tuple
    ortho_size: float
