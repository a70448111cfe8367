"""Box geometry and the θ-criterion (drop-in for ``fmm2d.geometry``).

These are the reference's host-side predicates (geometry.py:19-63), kept for
API compatibility and tests.  The engine never calls them: the device
connectivity kernels use the bit-exact restatement in csrc/common.cuh
(glibc hypot for radii, numpy's FMA cabs for distances, no contraction).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

DEFAULT_THETA = 0.5


@dataclass(frozen=True)
class Box:
    """Rectangle with complex center and half extents (geometry.py:19-29)."""

    center: complex | np.ndarray
    half_width: float | np.ndarray
    half_height: float | np.ndarray

    def radius(self):
        """Half-diagonal of the rectangle."""
        return np.hypot(self.half_width, self.half_height)


def _criterion(a: Box, b: Box, theta: float, swapped: bool):
    ra, rb = a.radius(), b.radius()
    d = np.abs(a.center - b.center)
    hi, lo = np.maximum(ra, rb), np.minimum(ra, rb)
    if swapped:
        hi, lo = lo, hi
    return hi + theta * lo <= theta * d


def well_separated(a: Box, b: Box, theta: float = DEFAULT_THETA):
    """max(r_a, r_b) + θ·min(r_a, r_b) <= θ·d (geometry.py:32-41)."""
    return _criterion(a, b, theta, swapped=False)


def well_separated_swapped(a: Box, b: Box, theta: float = DEFAULT_THETA):
    """min(r_a, r_b) + θ·max(r_a, r_b) <= θ·d (geometry.py:44-54)."""
    return _criterion(a, b, theta, swapped=True)


def split_direction(box: Box) -> str:
    """"y" if the box is taller than wide, else "x" (geometry.py:57-63)."""
    return "y" if box.half_height > box.half_width else "x"
