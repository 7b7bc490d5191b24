"""Oracle renumbering (TEST INFRASTRUCTURE ONLY).

Restates hodg/renumber.py: CSR adjacency (`from_edges`, :41-60), bandwidth
(:122-132), seeded shuffle (:117-119), Cuthill-McKee / RCM (:135-208, in C:
rcm_oracle.c), permutation application with the face re-sort (:211-269)
and the MatrixMarket spy export (:272-293).
"""

from __future__ import annotations

import numpy as np

from . import _clib
from .mesh import OMesh, Patch


class Graph:
    def __init__(self, n, indptr, indices):
        self.n, self.indptr, self.indices = n, indptr, indices

    @classmethod
    def from_edges(cls, n, edges):
        e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
        if e.size:
            if e.min() < 0 or e.max() >= n:
                raise ValueError("edge endpoint out of range")
            if np.any(e[:, 0] == e[:, 1]):
                raise ValueError("self-loop")
            u = np.minimum(e[:, 0], e[:, 1])
            v = np.maximum(e[:, 0], e[:, 1])
            uq = np.unique(np.stack([u, v], axis=1), axis=0)
            both = np.concatenate([uq, uq[:, ::-1]], axis=0)
        else:
            both = np.empty((0, 2), dtype=np.int64)
        both = both[np.lexsort((both[:, 1], both[:, 0]))]
        indptr = np.zeros(n + 1, dtype=np.int64)
        np.add.at(indptr, both[:, 0] + 1, 1)
        np.cumsum(indptr, out=indptr)
        return cls(n, indptr, np.ascontiguousarray(both[:, 1]))

    def degree(self):
        return np.diff(self.indptr)

    def edges(self):
        u = np.repeat(np.arange(self.n), self.degree())
        keep = u < self.indices
        return np.stack([u[keep], self.indices[keep]], axis=1)


def adjacency(mesh: OMesh) -> Graph:
    inner = mesh.face_cells[:, 1] >= 0
    return Graph.from_edges(mesh.n_cells, mesh.face_cells[inner])


def cuthill_mckee(g: Graph) -> np.ndarray:
    order = np.empty(g.n, dtype=np.int64)
    if g.n:
        rc = _clib.rcm_lib().ora_cuthill_mckee(g.n, _clib.ptr(g.indptr), _clib.ptr(g.indices), _clib.ptr(order))
        if rc != 0:
            raise MemoryError("oracle RCM allocation failed")
    return order


def rcm(g: Graph):
    """(forward, inverse): forward maps old -> new (hodg/renumber.py:203-208)."""
    order = cuthill_mckee(g)[::-1]
    fwd = np.empty(g.n, dtype=np.int64)
    fwd[order] = np.arange(g.n)
    return fwd, order.copy()


def random_permutation(n, seed=0):
    fwd = np.random.default_rng(seed).permutation(n).astype(np.int64)
    inv = np.empty(n, dtype=np.int64)
    inv[fwd] = np.arange(n)
    return fwd, inv


def bandwidth(g: Graph, fwd=None):
    e = g.edges()
    if e.shape[0] == 0:
        return 0
    if fwd is None:
        return int(np.max(np.abs(e[:, 0] - e[:, 1])))
    return int(np.max(np.abs(fwd[e[:, 0]] - fwd[e[:, 1]])))


def apply_permutation(m: OMesh, fwd, inv) -> OMesh:
    """hodg/renumber.py:211-269: cells reindexed, faces re-sorted by
    (min, max) incident new cell id then old face id."""
    l_new = fwd[m.face_cells[:, 0]]
    r_old = m.face_cells[:, 1]
    r_new = np.where(r_old >= 0, fwd[np.clip(r_old, 0, None)], l_new)
    forder = np.lexsort((np.arange(m.n_faces), np.maximum(l_new, r_new), np.minimum(l_new, r_new)))
    fmap = np.empty(m.n_faces, dtype=np.int64)
    fmap[forder] = np.arange(m.n_faces)
    fc = m.face_cells.copy()
    fc[:, 0] = fwd[m.face_cells[:, 0]]
    inner = m.face_cells[:, 1] >= 0
    fc[inner, 1] = fwd[m.face_cells[inner, 1]]
    fc = fc[forder].astype(np.int32)
    cf = np.where(m.cell_faces >= 0, fmap[np.clip(m.cell_faces, 0, None)], -1)[inv].astype(np.int32)
    cn = np.where(m.cell_neighbors >= 0, fwd[np.clip(m.cell_neighbors, 0, None)], -1)[inv].astype(np.int32)
    patches = [Patch(p.name, p.kind, np.sort(fmap[p.face_ids]).astype(np.int32)) for p in m.patches]
    return OMesh(m.dim, m.node_xy, m.cell_nodes[inv], m.cell_nfaces[inv], cf, m.cell_fsign[inv], cn,
                 m.cell_centroid[inv], m.cell_area[inv], m.cell_h[inv], m.face_nodes[forder], fc,
                 m.face_normal[forder], m.face_length[forder], m.face_patch[forder], patches)


def spy_text(g: Graph, fwd=None) -> str:
    n = g.n
    f = fwd if fwd is not None else np.arange(n, dtype=np.int64)
    e = g.edges()
    if e.shape[0]:
        pu, pv = f[e[:, 0]], f[e[:, 1]]
        rows = np.concatenate([np.arange(n, dtype=np.int64), pu, pv])
        cols = np.concatenate([np.arange(n, dtype=np.int64), pv, pu])
    else:
        rows = cols = np.arange(n, dtype=np.int64)
    o = np.lexsort((cols, rows))
    rows, cols = rows[o], cols[o]
    out = ["%%MatrixMarket matrix coordinate pattern symmetric", f"{n} {n} {rows.size}"]
    out += [f"{i + 1} {j + 1}" for i, j in zip(rows.tolist(), cols.tolist())]
    return "\n".join(out) + "\n"
