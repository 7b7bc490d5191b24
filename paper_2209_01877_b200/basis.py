"""Modal Taylor basis (`hodg/basis.py:1-69`) extended to 3D and order 3.

b_j = X^a Y^b (Z^c) with X = (x - xc)/h about the element centroid; 2D
h = sqrt(area) as in the reference, 3D h = cbrt(volume).  Modes are
degree-graded and, within a degree, ordered by descending x exponent then
descending y exponent -- the reference's `_EXPONENTS` order
(`hodg/basis.py:21`) extended.
"""

from __future__ import annotations

import numpy as np

__all__ = ["exponents", "n_basis", "NVAR"]

NVAR = {2: 4, 3: 5}


def exponents(dim: int, order: int) -> np.ndarray:
    out = []
    for d in range(order + 1):
        if dim == 2:
            for a in range(d, -1, -1):
                out.append((a, d - a))
        else:
            for a in range(d, -1, -1):
                for b in range(d - a, -1, -1):
                    out.append((a, b, d - a - b))
    return np.array(out, dtype=np.int64)


def n_basis(dim: int, order: int) -> int:
    return len(exponents(dim, order))
