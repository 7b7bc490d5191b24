"""Oracle meshes (TEST INFRASTRUCTURE ONLY).

2D: a restatement of the reference mesh builder (`hodg/mesh.py:177-425`):
face discovery by first traversal, shoelace area/centroid, CCW normals,
structured quad/tri generators and the seeded interior-node perturbation,
with the same floating-point expressions so geometry is bitwise equal to
the reference's (pinned by tests/test_oracle_golden.py).

3D: the tetrahedral analogue the reference does not have.  Each element's
vertices are stored in ascending node id; local face s is the face opposite
local vertex s, its vertices in ascending order.  Face ids follow first
traversal over (element, slot) exactly like the 2D builder; the unit
normal points out of the left (first-traversing) element.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

BC_KINDS = ("far_field", "slip_wall", "no_slip_wall")
TET_FACE_VERTS = np.array([[1, 2, 3], [0, 2, 3], [0, 1, 3], [0, 1, 2]], dtype=np.int64)


@dataclass
class Patch:
    name: str
    kind: str
    face_ids: np.ndarray


@dataclass
class OMesh:
    dim: int
    node_xy: np.ndarray  # (n_nodes, dim)
    cell_nodes: np.ndarray  # (N, 4) int32, -1 padded (2D triangles)
    cell_nfaces: np.ndarray  # (N,) int8
    cell_faces: np.ndarray  # (N, 4) int32
    cell_fsign: np.ndarray  # (N, 4) int8
    cell_neighbors: np.ndarray  # (N, 4) int32
    cell_centroid: np.ndarray  # (N, dim)
    cell_area: np.ndarray  # (N,) area (2D) / volume (3D)
    cell_h: np.ndarray  # (N,)
    face_nodes: np.ndarray  # (F, dim) int32
    face_cells: np.ndarray  # (F, 2) int32
    face_normal: np.ndarray  # (F, dim)
    face_length: np.ndarray  # (F,) length (2D) / area (3D)
    face_patch: np.ndarray  # (F,) int32
    patches: list = field(default_factory=list)

    @property
    def n_cells(self):
        return self.cell_nodes.shape[0]

    @property
    def n_faces(self):
        return self.face_nodes.shape[0]

    @property
    def n_nodes(self):
        return self.node_xy.shape[0]

    def bc_codes(self):
        codes = np.zeros(self.n_faces, dtype=np.int8)
        codes[self.face_cells[:, 1] < 0] = -1
        for p, patch in enumerate(self.patches):
            codes[self.face_patch == p] = BC_KINDS.index(patch.kind) + 1
        return codes


# ---------------------------------------------------------------------------
# 2D (restatement of hodg/mesh.py)

_EDGES = {3: ((0, 1), (1, 2), (2, 0)), 4: ((0, 1), (1, 2), (2, 3), (3, 0))}


def _shoelace(xy):
    # hodg/mesh.py:177-189
    x = xy[:, 0]
    y = xy[:, 1]
    xn = np.roll(x, -1)
    yn = np.roll(y, -1)
    cr = x * yn - xn * y
    area = 0.5 * np.sum(cr)
    if area == 0.0:
        return 0.0, xy.mean(axis=0)
    return float(area), np.array([np.sum((x + xn) * cr) / (6.0 * area), np.sum((y + yn) * cr) / (6.0 * area)])


def build_mesh_2d(node_xy, cells, patch_specs=None) -> OMesh:
    """hodg/mesh.py:192-333."""
    node_xy = np.ascontiguousarray(node_xy, dtype=np.float64)
    n = len(cells)
    cell_nodes = np.full((n, 4), -1, dtype=np.int32)
    nvert = np.zeros(n, dtype=np.int8)
    for c, nodes in enumerate(cells):
        cell_nodes[c, : len(nodes)] = nodes
        nvert[c] = len(nodes)
    area = np.empty(n)
    cen = np.empty((n, 2))
    for c in range(n):
        a, ce = _shoelace(node_xy[cell_nodes[c, : nvert[c]]])
        if a <= 0.0:
            raise ValueError(f"cell {c}: non-positive area")
        area[c] = a
        cen[c] = ce
    h = np.sqrt(area)
    keymap = {}
    fnodes, fcells = [], []
    cfaces = np.full((n, 4), -1, dtype=np.int32)
    csign = np.zeros((n, 4), dtype=np.int8)
    for c in range(n):
        for slot, (ea, eb) in enumerate(_EDGES[int(nvert[c])]):
            a = int(cell_nodes[c, ea])
            b = int(cell_nodes[c, eb])
            key = (min(a, b), max(a, b))
            fid = keymap.get(key)
            if fid is None:
                fid = len(fnodes)
                keymap[key] = fid
                fnodes.append((a, b))
                fcells.append([c, -1])
                csign[c, slot] = 1
            else:
                if fcells[fid][1] != -1:
                    raise ValueError("non-manifold face")
                fcells[fid][1] = c
                csign[c, slot] = -1
            cfaces[c, slot] = fid
    face_nodes = np.array(fnodes, dtype=np.int32)
    face_cells = np.array(fcells, dtype=np.int32)
    d = node_xy[face_nodes[:, 1]] - node_xy[face_nodes[:, 0]]
    flen = np.hypot(d[:, 0], d[:, 1])
    fnorm = np.column_stack([d[:, 1], -d[:, 0]]) / flen[:, None]
    neigh = np.full((n, 4), -1, dtype=np.int32)
    for c in range(n):
        for slot in range(nvert[c]):
            l, r = face_cells[cfaces[c, slot]]
            neigh[c, slot] = r if l == c else l
    fpatch = np.full(len(fnodes), -1, dtype=np.int32)
    patches = []
    for p, (name, kind, pairs) in enumerate(patch_specs or []):
        ids = []
        for a, b in pairs:
            fid = keymap[(min(a, b), max(a, b))]
            fpatch[fid] = p
            ids.append(fid)
        patches.append(Patch(name, kind, np.array(sorted(ids), dtype=np.int32)))
    return OMesh(2, node_xy, cell_nodes, nvert, cfaces, csign, neigh, cen, area, h,
                 face_nodes, face_cells, fnorm, flen, fpatch, patches)


def _grid(nx, ny, extent):
    x0, y0, x1, y1 = extent
    X, Y = np.meshgrid(np.linspace(x0, x1, nx + 1), np.linspace(y0, y1, ny + 1), indexing="xy")
    return np.column_stack([X.ravel(), Y.ravel()])


def _grid_sides(nx, ny, bc):
    bc = {s: bc for s in ("bottom", "right", "top", "left")} if isinstance(bc, str) else bc
    nid = lambda i, j: j * (nx + 1) + i  # noqa: E731
    sides = {
        "bottom": [(nid(i, 0), nid(i + 1, 0)) for i in range(nx)],
        "right": [(nid(nx, j), nid(nx, j + 1)) for j in range(ny)],
        "top": [(nid(i + 1, ny), nid(i, ny)) for i in range(nx)],
        "left": [(nid(0, j + 1), nid(0, j)) for j in range(ny)],
    }
    return [(s, bc[s], p) for s, p in sides.items()]


def quad_grid(nx, ny, extent=(0.0, 0.0, 1.0, 1.0), bc="far_field") -> OMesh:
    nid = lambda i, j: j * (nx + 1) + i  # noqa: E731
    cells = [(nid(i, j), nid(i + 1, j), nid(i + 1, j + 1), nid(i, j + 1)) for j in range(ny) for i in range(nx)]
    return build_mesh_2d(_grid(nx, ny, extent), cells, _grid_sides(nx, ny, bc))


def tri_grid(nx, ny, extent=(0.0, 0.0, 1.0, 1.0), bc="far_field") -> OMesh:
    nid = lambda i, j: j * (nx + 1) + i  # noqa: E731
    cells = []
    for j in range(ny):
        for i in range(nx):
            a, b, c, d = nid(i, j), nid(i + 1, j), nid(i + 1, j + 1), nid(i, j + 1)
            cells += [(a, b, c), (a, c, d)]
    return build_mesh_2d(_grid(nx, ny, extent), cells, _grid_sides(nx, ny, bc))


def perturb_2d(m: OMesh, amplitude, seed=0) -> OMesh:
    """hodg/mesh.py:396-425."""
    rng = np.random.default_rng(seed)
    bnodes = set(m.face_nodes[m.face_cells[:, 1] < 0].ravel().tolist())
    min_len = np.full(m.n_nodes, np.inf)
    for f in range(m.n_faces):
        a, b = m.face_nodes[f]
        min_len[a] = min(min_len[a], m.face_length[f])
        min_len[b] = min(min_len[b], m.face_length[f])
    xy = m.node_xy.copy()
    off = rng.uniform(-1.0, 1.0, size=xy.shape)
    for i in range(m.n_nodes):
        if i not in bnodes:
            xy[i] += amplitude * min_len[i] * off[i]
    cells = [tuple(m.cell_nodes[c, : m.cell_nfaces[c]]) for c in range(m.n_cells)]
    specs = [(p.name, p.kind, [tuple(m.face_nodes[f]) for f in p.face_ids]) for p in m.patches]
    return build_mesh_2d(xy, cells, specs)


# ---------------------------------------------------------------------------
# 3D tetrahedra


def build_tet_mesh(node_xyz, tets, patch_specs=None) -> OMesh:
    """Tetrahedral mesh from nodes, element->node lists and boundary
    patches (name, kind, [(a, b, c), ...])."""
    X = np.ascontiguousarray(node_xyz, dtype=np.float64)
    T = np.sort(np.asarray(tets, dtype=np.int64), axis=1)
    n = T.shape[0]
    V = X[T]  # (n, 4, 3)
    e1 = V[:, 1] - V[:, 0]
    e2 = V[:, 2] - V[:, 0]
    e3 = V[:, 3] - V[:, 0]
    det = (e1[:, 0] * (e2[:, 1] * e3[:, 2] - e2[:, 2] * e3[:, 1])
           - e1[:, 1] * (e2[:, 0] * e3[:, 2] - e2[:, 2] * e3[:, 0])
           + e1[:, 2] * (e2[:, 0] * e3[:, 1] - e2[:, 1] * e3[:, 0]))
    vol = np.abs(det) / 6.0
    if np.any(vol <= 0.0):
        raise ValueError("degenerate tetrahedron")
    cen = 0.25 * (V[:, 0] + V[:, 1] + V[:, 2] + V[:, 3])
    h = np.cbrt(vol)
    keys = T[:, TET_FACE_VERTS].reshape(-1, 3)  # (4n, 3), already ascending
    uniq, first, inv = np.unique(keys, axis=0, return_index=True, return_inverse=True)
    inv = inv.ravel()
    order = np.argsort(first, kind="stable")  # face ids by first traversal
    rank = np.empty_like(order)
    rank[order] = np.arange(order.size)
    fid_of_slot = rank[inv]  # (4n,)
    F = uniq.shape[0]
    counts = np.bincount(fid_of_slot, minlength=F)
    if counts.max() > 2:
        raise ValueError("non-manifold face")
    slot_ids = np.arange(4 * n)
    # first (left) and second (right) traversal of each face
    srt = np.lexsort((slot_ids, fid_of_slot))
    fs = fid_of_slot[srt]
    is_first = np.ones(4 * n, dtype=bool)
    is_first[1:] = fs[1:] != fs[:-1]
    left_slot = np.full(F, -1, dtype=np.int64)
    right_slot = np.full(F, -1, dtype=np.int64)
    left_slot[fs[is_first]] = srt[is_first]
    right_slot[fs[~is_first]] = srt[~is_first]
    face_cells = np.stack([left_slot // 4, np.where(right_slot >= 0, right_slot // 4, -1)], axis=1).astype(np.int32)
    face_nodes = uniq[order].astype(np.int32)
    cell_faces = fid_of_slot.reshape(n, 4).astype(np.int32)
    cell_fsign = np.where(np.isin(slot_ids, left_slot), 1, -1).reshape(n, 4).astype(np.int8)
    A = X[face_nodes[:, 0]]
    B = X[face_nodes[:, 1]]
    C = X[face_nodes[:, 2]]
    cr = np.cross(B - A, C - A)
    nrm = np.sqrt(cr[:, 0] * cr[:, 0] + cr[:, 1] * cr[:, 1] + cr[:, 2] * cr[:, 2])
    normal = cr / nrm[:, None]
    area = 0.5 * nrm
    # outward from the left element: compare with its vertex opposite the face
    lc = face_cells[:, 0]
    opp = X[T[lc, left_slot % 4]]
    flip = np.einsum("fd,fd->f", normal, A - opp) < 0.0
    normal[flip] *= -1.0
    neigh = np.empty((n, 4), dtype=np.int32)
    fc = face_cells[cell_faces]  # (n, 4, 2)
    me = np.arange(n)[:, None]
    neigh[:] = np.where(fc[..., 0] == me, fc[..., 1], fc[..., 0])
    fpatch = np.full(F, -1, dtype=np.int32)
    patches = []
    if patch_specs:
        lut = {tuple(k): i for i, k in enumerate(face_nodes.tolist())}
        for p, (name, kind, tris) in enumerate(patch_specs):
            ids = np.array([lut[tuple(sorted(t))] for t in tris], dtype=np.int64)
            if np.any(face_cells[ids, 1] >= 0):
                raise ValueError(f"patch {name}: interior face")
            fpatch[ids] = p
            patches.append(Patch(name, kind, np.sort(ids).astype(np.int32)))
    return OMesh(3, X, T.astype(np.int32), np.full(n, 4, dtype=np.int8), cell_faces, cell_fsign, neigh,
                 cen, vol, h, face_nodes, face_cells, normal, area, fpatch, patches)


# the 6 monotone paths 000 -> 111 through a unit cube (Kuhn / Freudenthal)
_KUHN_PATHS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]


def kuhn_box(n, extent=(0.0, 0.0, 0.0, 1.0, 1.0, 1.0), bc="far_field", ny=None, nz=None) -> OMesh:
    """n x ny x nz hexahedra, each split into 6 tetrahedra along the six
    monotone vertex paths; boundary patches xmin..zmax."""
    nx = n
    ny = n if ny is None else ny
    nz = n if nz is None else nz
    x0, y0, z0, x1, y1, z1 = extent
    xs = np.linspace(x0, x1, nx + 1)
    ys = np.linspace(y0, y1, ny + 1)
    zs = np.linspace(z0, z1, nz + 1)
    Z, Y, Xg = np.meshgrid(zs, ys, xs, indexing="ij")
    nodes = np.column_stack([Xg.ravel(), Y.ravel(), Z.ravel()])
    nid = lambda i, j, k: (k * (ny + 1) + j) * (nx + 1) + i  # noqa: E731
    I, J, K = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    I, J, K = (a.transpose(2, 1, 0).ravel() for a in (I, J, K))  # i fastest
    tets = []
    for path in _KUHN_PATHS:
        cur = np.zeros((I.size, 3), dtype=np.int64)
        verts = [nid(I, J, K)]
        for ax in path:
            cur[:, ax] += 1
            verts.append(nid(I + cur[:, 0], J + cur[:, 1], K + cur[:, 2]))
        tets.append(np.stack(verts, axis=1))
    tets = np.stack(tets, axis=1).reshape(-1, 4)  # hex-major, path-minor
    bc = {s: bc for s in ("xmin", "xmax", "ymin", "ymax", "zmin", "zmax")} if isinstance(bc, str) else bc
    specs = []
    for side in ("xmin", "xmax", "ymin", "ymax", "zmin", "zmax"):
        specs.append((side, bc[side], _box_side_tris(side, nx, ny, nz, nid)))
    return build_tet_mesh(nodes, tets, specs)


def _box_side_tris(side, nx, ny, nz, nid):
    """Boundary triangles of the Kuhn split on one box side: each boundary
    quad is cut along the diagonal joining its lowest and highest corner."""
    tris = []
    if side in ("xmin", "xmax"):
        i = 0 if side == "xmin" else nx
        for k in range(nz):
            for j in range(ny):
                a, b, c, d = nid(i, j, k), nid(i, j + 1, k), nid(i, j + 1, k + 1), nid(i, j, k + 1)
                tris += [(a, b, c), (a, c, d)]
    elif side in ("ymin", "ymax"):
        j = 0 if side == "ymin" else ny
        for k in range(nz):
            for i in range(nx):
                a, b, c, d = nid(i, j, k), nid(i + 1, j, k), nid(i + 1, j, k + 1), nid(i, j, k + 1)
                tris += [(a, b, c), (a, c, d)]
    else:
        k = 0 if side == "zmin" else nz
        for j in range(ny):
            for i in range(nx):
                a, b, c, d = nid(i, j, k), nid(i + 1, j, k), nid(i + 1, j + 1, k), nid(i, j + 1, k)
                tris += [(a, b, c), (a, c, d)]
    return tris


def perturb_3d(m: OMesh, amplitude, seed=3) -> OMesh:
    """Interior nodes moved by amplitude x (shortest incident face-edge
    length) x U(-1, 1)^3, the 3D analogue of hodg/mesh.py:396-425."""
    rng = np.random.default_rng(seed)
    bnodes = np.unique(m.face_nodes[m.face_cells[:, 1] < 0].ravel())
    T = m.cell_nodes.astype(np.int64)
    edges = T[:, [[0, 1], [0, 2], [0, 3], [1, 2], [1, 3], [2, 3]]].reshape(-1, 2)
    el = np.linalg.norm(m.node_xy[edges[:, 0]] - m.node_xy[edges[:, 1]], axis=1)
    min_len = np.full(m.n_nodes, np.inf)
    np.minimum.at(min_len, edges[:, 0], el)
    np.minimum.at(min_len, edges[:, 1], el)
    off = rng.uniform(-1.0, 1.0, size=m.node_xy.shape)
    xyz = m.node_xy.copy()
    interior = np.ones(m.n_nodes, dtype=bool)
    interior[bnodes] = False
    xyz[interior] += amplitude * min_len[interior, None] * off[interior]
    specs = [(p.name, p.kind, [tuple(m.face_nodes[f]) for f in p.face_ids]) for p in m.patches]
    return build_tet_mesh(xyz, m.cell_nodes, specs)
