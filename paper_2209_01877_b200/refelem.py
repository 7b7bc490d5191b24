"""Reference-element tables of the tetrahedral discretisation.

The device works in the monomial basis of the reference tetrahedron
    m_i(eta) = eta_1^a eta_2^b eta_3^c,  eta = xi - (1/4, 1/4, 1/4),
where x = V0 + J xi is the affine map of the element (vertices in ascending
node id).  The reference's physical Taylor basis b_j(X), X = (x - xc)/h
(`hodg/basis.py:1-69`) satisfies X = (J/h) eta, so each b_j is a fixed
combination of the m_i of the same degree; both span the same space and the
discrete operators coincide.  In this basis the per-cell tables of
`hodg/geometry.py:33-51` become element-independent constants (emitted for
the kernels by tools/gen_tables.py):

  VB[q, i]      m_i(eta_q)                     volume traces
  VD[q, i, d]   w_q dm_i/deta_d (eta_q)        volume integral, weight folded
  FB[s, q, i]   m_i(eta_{s,q})                 face traces on local face s
  FG[s, q, i]   wf_q m_i(eta_{s,q})            face gather, weight folded
  MINV          inverse reference mass matrix (exact rationals, rounded once)
  MEAN[i]       element mean of m_i            cell mean for the CFL dt
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction
from functools import lru_cache
from math import comb, factorial

import numpy as np

from .basis import exponents
from .quadrature import face_rule, volume_rule

TET_FACE_VERTS = ((1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2))


def _ref_moment(a, b, c) -> Fraction:
    """Mean over the unit tetrahedron (volume 1/6) of xi1^a xi2^b xi3^c."""
    return Fraction(6 * factorial(a) * factorial(b) * factorial(c), factorial(a + b + c + 3))


def centered_moment(alpha) -> Fraction:
    """Exact mean of prod_d (xi_d - 1/4)^alpha_d over the unit tetrahedron."""
    q = Fraction(-1, 4)
    tot = Fraction(0)
    a0, a1, a2 = (int(a) for a in alpha)
    for i in range(a0 + 1):
        for j in range(a1 + 1):
            for k in range(a2 + 1):
                tot += comb(a0, i) * comb(a1, j) * comb(a2, k) * q ** (a0 - i + a1 - j + a2 - k) * _ref_moment(i, j, k)
    return tot


def monomials(E, eta):
    out = np.ones(eta.shape[:-1] + (len(E),))
    for j, e in enumerate(E):
        for d in range(3):
            if e[d]:
                out[..., j] *= eta[..., d] ** e[d]
    return out


def _exact_inverse(M):
    """Gauss-Jordan inverse over the rationals."""
    n = len(M)
    A = [list(row) + [Fraction(int(i == j)) for j in range(n)] for i, row in enumerate(M)]
    for c in range(n):
        piv = next(r for r in range(c, n) if A[r][c] != 0)
        A[c], A[piv] = A[piv], A[c]
        pv = A[c][c]
        A[c] = [x / pv for x in A[c]]
        for r in range(n):
            if r != c and A[r][c] != 0:
                f = A[r][c]
                A[r] = [x - f * y for x, y in zip(A[r], A[c])]
    return [row[n:] for row in A]


@dataclass(frozen=True)
class RefTables:
    order: int
    E: np.ndarray
    vol_points: np.ndarray  # (nqv, 4) barycentric
    vol_weights: np.ndarray  # (nqv,) sum 1
    face_points: np.ndarray  # (nqf, 3) barycentric
    face_weights: np.ndarray  # (nqf,) sum 1
    VB: np.ndarray
    VD: np.ndarray
    FB: np.ndarray
    FG: np.ndarray
    MINV: np.ndarray
    MEAN: np.ndarray

    @property
    def nb(self):
        return len(self.E)

    @property
    def nqv(self):
        return len(self.vol_weights)

    @property
    def nqf(self):
        return len(self.face_weights)

    @property
    def projector(self) -> np.ndarray:
        """(nb, nqv): L2 projection of volume-point values onto m_i."""
        return self.MINV @ (self.VB * self.vol_weights[:, None]).T


@lru_cache(maxsize=None)
def ref_tables(order: int) -> RefTables:
    E = exponents(3, order)
    nb = len(E)
    bary, w = volume_rule(order, 3)
    eta = bary[:, 1:4] - 0.25
    VB = monomials(E, eta)
    VD = np.zeros((len(w), nb, 3))
    for i, e in enumerate(E):
        for d in range(3):
            if e[d] == 0:
                continue
            ee = np.array(e)
            ee[d] -= 1
            VD[:, i, d] = w * e[d] * monomials(ee[None, :], eta)[:, 0]
    fb, fw = face_rule(order, 3)
    FB = np.zeros((4, len(fw), nb))
    for s, verts in enumerate(TET_FACE_VERTS):
        xi = np.zeros((len(fw), 3))
        for j, vtx in enumerate(verts):
            if vtx > 0:
                xi[:, vtx - 1] += fb[:, j]
        FB[s] = monomials(E, xi - 0.25)
    FG = FB * fw[None, :, None]
    Mx = [[centered_moment(E[i] + E[k]) for k in range(nb)] for i in range(nb)]
    MINV = np.array([[float(x) for x in row] for row in _exact_inverse(Mx)])
    MEAN = np.array([float(centered_moment(e)) for e in E])
    return RefTables(order, E, bary, w, fb, fw, VB, VD, FB, FG, MINV, MEAN)
