"""Oracle geometry tables (TEST INFRASTRUCTURE ONLY).

Restates `hodg/geometry.py:33-220`: per-element quadrature points and
physical weights, Taylor-basis values and gradients at those points, per-
face basis traces, mass matrices and their inverses (`np.linalg.inv`), and
basis means.  The 2D path loops per cell with the reference's own numpy
expressions so tables are bitwise equal to the reference's; the 3D path is
the same table-driven discretisation vectorised over tetrahedra.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_2209_01877_b200.basis import exponents
from paper_2209_01877_b200.quadrature import face_rule, gauss_legendre_1d, tet_rule, triangle_rule


@dataclass
class OTables:
    order: int
    n_basis: int
    vol_xy: np.ndarray
    vol_w: np.ndarray
    vol_basis: np.ndarray
    vol_grad: np.ndarray  # (dim, N, nqv, nb)
    face_xy: np.ndarray
    face_w: np.ndarray
    face_basis_l: np.ndarray
    face_basis_r: np.ndarray
    mass: np.ndarray
    minv: np.ndarray
    basis_mean: np.ndarray

    @property
    def n_vol_points(self):
        return self.vol_w.shape[1]

    @property
    def n_face_points(self):
        return self.face_w.shape[1]

    def cast(self, dtype):
        """Float tables at kernel precision (hodg/geometry.py:82-95)."""
        names = ("vol_w", "vol_basis", "vol_grad", "face_w", "face_basis_l", "face_basis_r")
        return {n: np.ascontiguousarray(getattr(self, n), dtype=dtype) for n in names}


def _values(E, pts, cen, h):
    """hodg/basis.py:40-51 with the same per-mode expression."""
    rel = [(pts[..., d] - cen[..., d]) / h for d in range(pts.shape[-1])]
    out = np.empty(pts.shape[:-1] + (len(E),))
    for j in range(len(E)):
        v = rel[0] ** E[j, 0]
        for d in range(1, pts.shape[-1]):
            v = v * rel[d] ** E[j, d]
        out[..., j] = v
    return out


def _gradients(E, pts, cen, h):
    """hodg/basis.py:53-69: d/dx_d b_j = a_d X_d^(a_d - 1) * rest / h."""
    dim = pts.shape[-1]
    rel = [(pts[..., d] - cen[..., d]) / h for d in range(dim)]
    out = np.zeros((dim,) + pts.shape[:-1] + (len(E),))
    for j in range(len(E)):
        for d in range(dim):
            a = E[j, d]
            if a == 0:
                continue
            v = a
            for e in range(dim):  # reference order: (a * X^..) * Y^.. / h
                v = v * rel[e] ** (E[j, e] - (1 if e == d else 0))
            out[d, ..., j] = v / h
    return out


def _quad_map(corners, ref):
    # hodg/geometry.py:98-117
    xi = ref[:, 0]
    eta = ref[:, 1]
    shape = 0.25 * np.column_stack([(1 - xi) * (1 - eta), (1 + xi) * (1 - eta), (1 + xi) * (1 + eta), (1 - xi) * (1 + eta)])
    dxi = 0.25 * np.column_stack([-(1 - eta), (1 - eta), (1 + eta), -(1 + eta)])
    deta = 0.25 * np.column_stack([-(1 - xi), -(1 + xi), (1 + xi), (1 - xi)])
    xy = shape @ corners
    jx = dxi @ corners
    jy = deta @ corners
    return xy, jx[:, 0] * jy[:, 1] - jx[:, 1] * jy[:, 0]


def tables_2d(mesh, order) -> OTables:
    """hodg/geometry.py:120-220, per-cell loop."""
    E = exponents(2, order)
    nb = len(E)
    n = mesh.n_cells
    tri_b, tri_w = triangle_rule(max(2 * order, 1))
    g1, gw = gauss_legendre_1d(order + 1)
    Xi, Eta = np.meshgrid(g1, g1, indexing="ij")
    quad_p = np.column_stack([Xi.ravel(), Eta.ravel()])
    quad_w = np.outer(gw, gw).ravel()
    nqv = max(tri_w.size if np.any(mesh.cell_nfaces == 3) else 0,
              quad_w.size if np.any(mesh.cell_nfaces == 4) else 0)
    vol_xy = np.zeros((n, nqv, 2))
    vol_w = np.zeros((n, nqv))
    vol_b = np.zeros((n, nqv, nb))
    vol_g = np.zeros((2, n, nqv, nb))
    mass = np.zeros((n, nb, nb))
    minv = np.zeros((n, nb, nb))
    bmean = np.zeros((n, nb))
    for c in range(n):
        nv = int(mesh.cell_nfaces[c])
        corners = mesh.node_xy[mesh.cell_nodes[c, :nv]]
        if nv == 3:
            xy = tri_b @ corners
            w = tri_w * mesh.cell_area[c]
        else:
            xy, det = _quad_map(corners, quad_p)
            w = quad_w * det
        nq = xy.shape[0]
        cen = mesh.cell_centroid[c]
        h = mesh.cell_h[c]
        b = _values(E, xy, cen, h)
        g = _gradients(E, xy, cen, h)
        vol_xy[c, :nq] = xy
        vol_w[c, :nq] = w
        vol_b[c, :nq] = b
        vol_g[:, c, :nq] = g
        m = np.einsum("q,qj,qk->jk", w, b, b)
        mass[c] = m
        minv[c] = np.linalg.inv(m)
        bmean[c] = (w @ b) / mesh.cell_area[c]
    nqf = order + 1
    t1d, w1d = gauss_legendre_1d(nqf)
    nf = mesh.n_faces
    face_xy = np.zeros((nf, nqf, 2))
    face_w = np.zeros((nf, nqf))
    a_xy = mesh.node_xy[mesh.face_nodes[:, 0]]
    b_xy = mesh.node_xy[mesh.face_nodes[:, 1]]
    for q in range(nqf):
        s = 0.5 * (1.0 + t1d[q])
        face_xy[:, q, :] = a_xy + s * (b_xy - a_xy)
        face_w[:, q] = 0.5 * w1d[q] * mesh.face_length
    fbl = np.zeros((nf, nqf, nb))
    fbr = np.zeros((nf, nqf, nb))
    for f in range(nf):
        for side, cell in enumerate(mesh.face_cells[f]):
            if cell < 0:
                continue
            vals = _values(E, face_xy[f], mesh.cell_centroid[cell], mesh.cell_h[cell])
            (fbl if side == 0 else fbr)[f] = vals
    return OTables(order, nb, vol_xy, vol_w, vol_b, vol_g, face_xy, face_w, fbl, fbr, mass, minv, bmean)


def tables_3d(mesh, order) -> OTables:
    """The 3D analogue, vectorised over tetrahedra (affine elements)."""
    E = exponents(3, order)
    nb = len(E)
    bary, wq = tet_rule(max(2 * order, 1))
    V = mesh.node_xy[mesh.cell_nodes.astype(np.int64)]  # (N, 4, 3)
    xy = (bary[None, :, 0, None] * V[:, None, 0] + bary[None, :, 1, None] * V[:, None, 1]
          + bary[None, :, 2, None] * V[:, None, 2] + bary[None, :, 3, None] * V[:, None, 3])
    cen = mesh.cell_centroid[:, None, :]
    h = mesh.cell_h[:, None]
    w = wq[None, :] * mesh.cell_area[:, None]
    b = _values(E, xy, cen, h)
    g = _gradients(E, xy, cen, h)
    mass = np.einsum("cq,cqj,cqk->cjk", w, b, b)
    minv = np.linalg.inv(mass)
    bmean = np.einsum("cq,cqj->cj", w, b) / mesh.cell_area[:, None]
    fb, fw = face_rule(order, 3)
    P = mesh.node_xy[mesh.face_nodes.astype(np.int64)]  # (F, 3, 3)
    fxy = (fb[None, :, 0, None] * P[:, None, 0] + fb[None, :, 1, None] * P[:, None, 1]
           + fb[None, :, 2, None] * P[:, None, 2])
    face_w = fw[None, :] * mesh.face_length[:, None]
    L = mesh.face_cells[:, 0].astype(np.int64)
    R = mesh.face_cells[:, 1].astype(np.int64)
    fbl = _values(E, fxy, mesh.cell_centroid[L][:, None, :], mesh.cell_h[L][:, None])
    Rc = np.where(R >= 0, R, 0)
    fbr = _values(E, fxy, mesh.cell_centroid[Rc][:, None, :], mesh.cell_h[Rc][:, None])
    fbr[R < 0] = 0.0
    return OTables(order, nb, xy, w, b, g, fxy, face_w, fbl, fbr, mass, minv, bmean)


def compute_tables(mesh, order) -> OTables:
    return tables_3d(mesh, order) if mesh.dim == 3 else tables_2d(mesh, order)
