"""Unstructured tetrahedral meshes: flat arrays indexed by entity id, the 3D
analogue of the reference's `hodg/mesh.py` (Mesh arrays :97-174, face
discovery :241-286, generators :361-393, perturbation :396-425, HODG-MESH
text format :431-560, validation :566-629).

Conventions (the device kernels rely on them):
  * each element's four node ids are stored ascending; local face s is the
    face opposite local vertex s, its vertices in ascending order -- so the
    two elements sharing a face enumerate its vertices (and, the face rules
    being fully symmetric, its quadrature points) identically;
  * face ids follow the first traversal over (element, slot), the first
    traverser is the left element, the unit normal points left -> right
    (outward at boundaries), as in the reference's 2D builder;
  * `cell_area` holds element volumes and `face_length` face areas, keeping
    the reference's field names.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "BC_KINDS",
    "MeshError",
    "MeshParseError",
    "TopologyError",
    "BoundaryPatch",
    "TetMesh",
    "build_tet_mesh",
    "generate_tet_box",
    "perturb_interior_nodes",
    "save_mesh",
    "load_mesh",
    "validate",
]

BC_KINDS = ("far_field", "slip_wall", "no_slip_wall")
FACE_LOCAL = np.array([[1, 2, 3], [0, 2, 3], [0, 1, 3], [0, 1, 2]], dtype=np.int64)


class MeshError(Exception):
    pass


class MeshParseError(MeshError):
    def __init__(self, path, line_no, message):
        super().__init__(f"{path}:{line_no}: {message}")
        self.line_no = line_no


class TopologyError(MeshError):
    pass


@dataclass(frozen=True)
class BoundaryPatch:
    name: str
    kind: str
    face_ids: np.ndarray

    def __post_init__(self):
        if self.kind not in BC_KINDS:
            raise MeshError(f"unknown boundary kind {self.kind!r}")


@dataclass
class TetMesh:
    node_xy: np.ndarray  # (n_nodes, 3)
    cell_nodes: np.ndarray  # (N, 4) int32 ascending
    cell_faces: np.ndarray  # (N, 4) int32, slot s = face opposite vertex s
    cell_fsign: np.ndarray  # (N, 4) int8: +1 left, -1 right
    cell_neighbors: np.ndarray  # (N, 4) int32, -1 at boundary
    cell_centroid: np.ndarray  # (N, 3)
    cell_area: np.ndarray  # (N,) volume
    cell_h: np.ndarray  # (N,) cbrt(volume)
    face_nodes: np.ndarray  # (F, 3) int32 ascending
    face_cells: np.ndarray  # (F, 2) int32, right = -1 at boundary
    face_slots: np.ndarray  # (F, 2) int8, local slot in left / right element (-1)
    face_normal: np.ndarray  # (F, 3) unit, left -> right
    face_length: np.ndarray  # (F,) area
    face_patch: np.ndarray  # (F,) int32 patch index or -1
    patches: list = field(default_factory=list)

    dim = 3

    @property
    def n_nodes(self) -> int:
        return self.node_xy.shape[0]

    @property
    def n_cells(self) -> int:
        return self.cell_nodes.shape[0]

    @property
    def n_faces(self) -> int:
        return self.face_nodes.shape[0]

    @property
    def n_interior_faces(self) -> int:
        return int(np.count_nonzero(self.face_cells[:, 1] >= 0))

    @property
    def cell_nvert(self) -> np.ndarray:
        return np.full(self.n_cells, 4, dtype=np.int8)

    def boundary_kind_codes(self) -> np.ndarray:
        """0 interior, 1 far_field, 2 slip_wall, 3 no_slip_wall, -1 unpatched
        boundary (hodg/mesh.py:166-174)."""
        codes = np.zeros(self.n_faces, dtype=np.int8)
        codes[self.face_cells[:, 1] < 0] = -1
        for p, patch in enumerate(self.patches):
            codes[self.face_patch == p] = BC_KINDS.index(patch.kind) + 1
        return codes

    def raw(self):
        """(nodes, elements, patch specs) that rebuild this mesh."""
        specs = [(p.name, p.kind, [tuple(int(x) for x in self.face_nodes[f]) for f in p.face_ids])
                 for p in self.patches]
        return self.node_xy, self.cell_nodes, specs


def _signed_volume6(V):
    a = V[:, 1] - V[:, 0]
    b = V[:, 2] - V[:, 0]
    c = V[:, 3] - V[:, 0]
    return np.einsum("nd,nd->n", a, np.cross(b, c))


def build_tet_mesh(node_xyz, tets, patch_specs=None, device=None) -> TetMesh:
    """Assemble a tetrahedral mesh from nodes, element->node lists and
    boundary patches [(name, kind, [(a, b, c), ...]), ...].  With `device`
    (e.g. "cuda") the connectivity and geometry are built on the GPU
    (`hodg_mesh_setup`, csrc/setup.cu): identical integer arrays, float
    geometry equal up to libm-vs-CUDA rounding of the element size h."""
    X = np.ascontiguousarray(node_xyz, dtype=np.float64)
    if X.ndim != 2 or X.shape[1] != 3:
        raise MeshError("node coordinates must be an (n, 3) array")
    if not np.all(np.isfinite(X)):
        raise TopologyError("non-finite node coordinates")
    T = np.asarray(tets, dtype=np.int64)
    if T.ndim != 2 or T.shape[1] != 4 or T.shape[0] == 0:
        raise MeshError("elements must be a non-empty (N, 4) array")
    if T.min() < 0 or T.max() >= X.shape[0]:
        raise TopologyError("element node index out of range")
    T = np.sort(T, axis=1)
    if np.any(T[:, 1:] == T[:, :-1]):
        raise TopologyError("element with a repeated node")
    n = T.shape[0]
    nn = np.int64(X.shape[0])
    if device is not None:
        (face_cells, face_slots, face_nodes, normal, area, cell_faces, cell_fsign, cell_neighbors, vol, centroid,
         h) = _setup_on_device(X, T, device)
        F = face_cells.shape[0]
        return _with_patches(X, T, patch_specs, nn, F, face_nodes, face_cells, cell_faces, cell_fsign,
                             cell_neighbors, centroid, vol, h, face_slots, normal, area)
    V = X[T]
    vol = np.abs(_signed_volume6(V)) / 6.0
    if np.any(vol <= 0.0):
        raise TopologyError(f"element {int(np.argmin(vol))}: degenerate (zero volume)")
    centroid = 0.25 * (V[:, 0] + V[:, 1] + V[:, 2] + V[:, 3])
    h = np.cbrt(vol)

    # face discovery: pack the ascending triple into one 64-bit key
    tri = T[:, FACE_LOCAL].reshape(-1, 3)  # (4n, 3), slot-major within element
    key = (tri[:, 0] * nn + tri[:, 1]) * nn + tri[:, 2]
    order = np.argsort(key, kind="stable")  # ties keep traversal order
    ks = key[order]
    new_run = np.empty(ks.size, dtype=bool)
    new_run[0] = True
    new_run[1:] = ks[1:] != ks[:-1]
    run_id = np.cumsum(new_run) - 1
    run_start = np.flatnonzero(new_run)
    run_len = np.diff(np.append(run_start, ks.size))
    if run_len.max() > 2:
        raise TopologyError("face shared by more than two elements (non-manifold)")
    first_slot = order[run_start]  # first traversal of each distinct face
    face_rank = np.empty(run_start.size, dtype=np.int64)
    face_rank[np.argsort(first_slot, kind="stable")] = np.arange(run_start.size)
    slot_face = np.empty(4 * n, dtype=np.int64)
    slot_face[order] = face_rank[run_id]
    F = run_start.size
    left_slot = np.empty(F, dtype=np.int64)
    left_slot[face_rank] = first_slot
    right_slot = np.full(F, -1, dtype=np.int64)
    two = run_len == 2
    right_slot[face_rank[two]] = order[run_start[two] + 1]

    face_cells = np.stack([left_slot // 4, np.where(right_slot >= 0, right_slot // 4, -1)], axis=1).astype(np.int32)
    face_slots = np.stack([left_slot % 4, np.where(right_slot >= 0, right_slot % 4, -1)], axis=1).astype(np.int8)
    face_nodes = tri[left_slot].astype(np.int32)
    cell_faces = slot_face.reshape(n, 4).astype(np.int32)
    sign = np.full(4 * n, -1, dtype=np.int8)
    sign[left_slot] = 1
    cell_fsign = sign.reshape(n, 4)

    A = X[face_nodes[:, 0]]
    cr = np.cross(X[face_nodes[:, 1]] - A, X[face_nodes[:, 2]] - A)
    norm = np.sqrt(np.einsum("fd,fd->f", cr, cr))
    if np.any(norm <= 0.0):
        raise TopologyError("zero-area face")
    normal = cr / norm[:, None]
    opp = X[T[face_cells[:, 0], face_slots[:, 0]]]  # left element's vertex opposite the face
    inward = np.einsum("fd,fd->f", normal, A - opp) < 0.0
    normal[inward] = -normal[inward]
    area = 0.5 * norm

    fc = face_cells[cell_faces]
    cell_neighbors = np.where(fc[..., 0] == np.arange(n)[:, None], fc[..., 1], fc[..., 0]).astype(np.int32)
    return _with_patches(X, T, patch_specs, nn, F, face_nodes, face_cells, cell_faces, cell_fsign, cell_neighbors,
                         centroid, vol, h, face_slots, normal, area)


def _setup_on_device(X, T, device):
    """hodg_mesh_setup: connectivity + geometry on the GPU, copied back."""
    import torch

    from . import _lib

    L = _lib.lib()
    n = T.shape[0]
    dev = torch.device(device)
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    Xd, Td = up(X), up(T.astype(np.int32))
    cap = 4 * n
    e = lambda shape, dt: torch.empty(shape, dtype=dt, device=dev)  # noqa: E731
    out = [e((cap, 2), torch.int32), e((cap, 2), torch.int8), e((cap, 3), torch.int32), e((cap, 3), torch.float64),
           e(cap, torch.float64), e((n, 4), torch.int32), e((n, 4), torch.int8), e((n, 4), torch.int32),
           e(n, torch.float64), e((n, 3), torch.float64), e(n, torch.float64)]
    wb = int(L.hodg_mesh_setup_work_bytes(n))
    if wb < 0:
        raise MeshError("mesh too large for the device setup")
    work = e(wb, torch.uint8)
    nf = np.zeros(1, dtype=np.int64)
    rc = L.hodg_mesh_setup(X.shape[0], n, _lib.ptr(Xd), _lib.ptr(Td), *[_lib.ptr(t) for t in out], nf.ctypes.data,
                           _lib.ptr(work), _lib.stream_ptr())
    if rc == 5:  # HODG_ETOPOLOGY
        raise TopologyError({-1: "face shared by more than two elements (non-manifold)", -2: "zero-area face",
                             -3: "degenerate element (zero volume)"}.get(int(nf[0]), "invalid topology"))
    _lib.check(rc, "hodg_mesh_setup")
    F = int(nf[0])
    fc, fs, fn, nrm, area, cf, cs, cn, vol, cen, h = [t.cpu().numpy() for t in out]
    return fc[:F], fs[:F], fn[:F], nrm[:F], area[:F], cf, cs, cn, vol, cen, h


def _with_patches(X, T, patch_specs, nn, F, face_nodes, face_cells, cell_faces, cell_fsign, cell_neighbors,
                  centroid, vol, h, face_slots, normal, area) -> TetMesh:
    face_patch = np.full(F, -1, dtype=np.int32)
    patches = []
    if patch_specs:
        fkey = (face_nodes[:, 0].astype(np.int64) * nn + face_nodes[:, 1]) * nn + face_nodes[:, 2]
        srt = np.argsort(fkey)
        for p, (name, kind, tris) in enumerate(patch_specs):
            t3 = np.sort(np.asarray(tris, dtype=np.int64).reshape(-1, 3), axis=1)
            k = (t3[:, 0] * nn + t3[:, 1]) * nn + t3[:, 2]
            pos = np.searchsorted(fkey[srt], k)
            ok = (pos < F) & (fkey[srt][np.minimum(pos, F - 1)] == k)
            if not np.all(ok):
                raise TopologyError(f"patch {name!r}: no face with nodes {t3[~ok][0].tolist()}")
            ids = srt[pos]
            if np.any(face_cells[ids, 1] >= 0):
                raise TopologyError(f"patch {name!r}: interior face")
            if np.any(face_patch[ids] != -1):
                raise TopologyError(f"patch {name!r}: face already in another patch")
            face_patch[ids] = p
            patches.append(BoundaryPatch(name, kind, np.sort(ids).astype(np.int32)))

    return TetMesh(X, T.astype(np.int32), cell_faces, cell_fsign, cell_neighbors, centroid, vol, h,
                   face_nodes, face_cells, face_slots, normal, area, face_patch, patches)


# six monotone lattice paths 000 -> 111 (Kuhn / Freudenthal split)
_PATHS = ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0))
_SIDES = ("xmin", "xmax", "ymin", "ymax", "zmin", "zmax")


def generate_tet_box(nx: int, ny: int | None = None, nz: int | None = None,
                     extent=(0.0, 0.0, 0.0, 1.0, 1.0, 1.0), bc="far_field", device=None) -> TetMesh:
    """Structured hexahedral lattice, each hex split into six tetrahedra
    along its main diagonal (conforming; 6 nx ny nz elements).  `bc` is one
    kind or a dict keyed by xmin..zmax.  Elements are numbered hex-major
    (x fastest), path-minor."""
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    if min(nx, ny, nz) < 1:
        raise MeshError("box dimensions must be at least 1")
    x0, y0, z0, x1, y1, z1 = extent
    gx, gy, gz = np.linspace(x0, x1, nx + 1), np.linspace(y0, y1, ny + 1), np.linspace(z0, z1, nz + 1)
    nodes = np.stack(np.meshgrid(gx, gy, gz, indexing="ij"), axis=-1).transpose(2, 1, 0, 3).reshape(-1, 3)

    def nid(i, j, k):
        return (k * (ny + 1) + j) * (nx + 1) + i

    k3, j3, i3 = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    i3, j3, k3 = i3.ravel(), j3.ravel(), k3.ravel()
    elems = np.empty((i3.size, 6, 4), dtype=np.int64)
    for p, path in enumerate(_PATHS):
        off = np.zeros(3, dtype=np.int64)
        elems[:, p, 0] = nid(i3, j3, k3)
        for s, ax in enumerate(path):
            off[ax] += 1
            elems[:, p, s + 1] = nid(i3 + off[0], j3 + off[1], k3 + off[2])
    kinds = {s: bc for s in _SIDES} if isinstance(bc, str) else dict(bc)
    specs = []
    for side in _SIDES:
        axis = "xyz".index(side[0])
        fixed = 0 if side.endswith("min") else (nx, ny, nz)[axis]
        u_ax, w_ax = [a for a in range(3) if a != axis]
        nu, nw = (nx, ny, nz)[u_ax], (nx, ny, nz)[w_ax]
        uu, ww = np.meshgrid(np.arange(nu), np.arange(nw), indexing="ij")
        uu, ww = uu.ravel(), ww.ravel()

        def corner(du, dw):
            idx = [None, None, None]
            idx[axis] = np.full(uu.size, fixed)
            idx[u_ax] = uu + du
            idx[w_ax] = ww + dw
            return nid(*idx)

        lo, hi = corner(0, 0), corner(1, 1)
        tris = np.concatenate([np.stack([lo, corner(1, 0), hi], axis=1), np.stack([lo, corner(0, 1), hi], axis=1)])
        specs.append((side, kinds[side], tris))
    return build_tet_mesh(nodes, elems.reshape(-1, 4), specs, device=device)


def generate_wing_box(n: int, sweep_deg: float = 30.0, span: float = 0.6, root_chord: float = 0.35,
                      taper: float = 0.56, thickness: float = 0.10, device=None) -> TetMesh:
    """BASELINE config 4's synthetic ONERA-M6-like geometry:
    the Kuhn-split unit cube of n^3 hexahedra with a swept, tapered
    diamond-section wedge wing cut out -- hexahedra whose centre lies inside
    the wing are removed (a lattice-conforming, staircase surface).  The wing
    root sits on the z = 0 symmetry plane (slip wall), its leading edge at
    x = 0.3 + z tan(sweep), chord root_chord (1 - (1 - taper) z / span),
    half-thickness `thickness` x chord x min(xi / 0.3, (1 - xi) / 0.7) about
    y = 0.5.  Boundaries: wing surface `wing` (slip wall), z = 0 `symmetry`
    (slip wall), the other five sides far field."""
    if n < 4:
        raise MeshError("wing box needs n >= 4")
    g = np.linspace(0.0, 1.0, n + 1)
    nodes = np.stack(np.meshgrid(g, g, g, indexing="ij"), axis=-1).transpose(2, 1, 0, 3).reshape(-1, 3)

    def nid(i, j, k):
        return (k * (n + 1) + j) * (n + 1) + i

    k3, j3, i3 = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    i3, j3, k3 = i3.ravel(), j3.ravel(), k3.ravel()
    xc, yc, zc = (i3 + 0.5) / n, (j3 + 0.5) / n, (k3 + 0.5) / n
    chord = root_chord * (1.0 - (1.0 - taper) * zc / span)
    xi = (xc - (0.3 + zc * np.tan(np.deg2rad(sweep_deg)))) / chord
    half = thickness * chord * np.minimum(xi / 0.3, (1.0 - xi) / 0.7)
    inside = (zc <= span) & (xi >= 0.0) & (xi <= 1.0) & (np.abs(yc - 0.5) <= half)
    keep = ~inside
    i3, j3, k3 = i3[keep], j3[keep], k3[keep]
    elems = np.empty((i3.size, 6, 4), dtype=np.int64)
    for p, path in enumerate(_PATHS):
        off = np.zeros(3, dtype=np.int64)
        elems[:, p, 0] = nid(i3, j3, k3)
        for s_, ax in enumerate(path):
            off[ax] += 1
            elems[:, p, s_ + 1] = nid(i3 + off[0], j3 + off[1], k3 + off[2])
    # unreferenced nodes (strictly inside the wing) are dropped
    used = np.unique(elems)
    remap = np.full(nodes.shape[0], -1, dtype=np.int64)
    remap[used] = np.arange(used.size)
    m = build_tet_mesh(nodes[used], remap[elems.reshape(-1, 4)], None, device=device)
    bnd = np.flatnonzero(m.face_cells[:, 1] < 0)
    X = m.node_xy[m.face_nodes[bnd].astype(np.int64)]
    eps = 1e-12
    on = lambda d, v: np.all(np.abs(X[:, :, d] - v) < eps, axis=1)  # noqa: E731
    sym = on(2, 0.0)
    outer = on(0, 0.0) | on(0, 1.0) | on(1, 0.0) | on(1, 1.0) | on(2, 1.0)
    wing = ~(sym | outer)
    face_patch = np.full(m.n_faces, -1, dtype=np.int32)
    patches = []
    for p, (name, kind, sel) in enumerate((("far", "far_field", outer), ("symmetry", "slip_wall", sym),
                                            ("wing", "slip_wall", wing))):
        ids = np.sort(bnd[sel]).astype(np.int32)
        face_patch[ids] = p
        patches.append(BoundaryPatch(name, kind, ids))
    return TetMesh(m.node_xy, m.cell_nodes, m.cell_faces, m.cell_fsign, m.cell_neighbors, m.cell_centroid,
                   m.cell_area, m.cell_h, m.face_nodes, m.face_cells, m.face_slots, m.face_normal, m.face_length,
                   face_patch, patches)


def perturb_interior_nodes(mesh: TetMesh, amplitude: float, seed: int = 0) -> TetMesh:
    """Interior nodes moved by amplitude x (shortest incident edge) x
    U(-1, 1)^3; boundary nodes fixed, patches preserved (3D analogue of
    hodg/mesh.py:396-425)."""
    rng = np.random.default_rng(seed)
    X = mesh.node_xy
    T = mesh.cell_nodes.astype(np.int64)
    e = T[:, [[0, 1], [0, 2], [0, 3], [1, 2], [1, 3], [2, 3]]].reshape(-1, 2)
    length = np.linalg.norm(X[e[:, 0]] - X[e[:, 1]], axis=1)
    shortest = np.full(mesh.n_nodes, np.inf)
    np.minimum.at(shortest, e[:, 0], length)
    np.minimum.at(shortest, e[:, 1], length)
    offsets = rng.uniform(-1.0, 1.0, size=X.shape)
    movable = np.ones(mesh.n_nodes, dtype=bool)
    movable[np.unique(mesh.face_nodes[mesh.face_cells[:, 1] < 0])] = False
    Y = X.copy()
    Y[movable] += amplitude * shortest[movable, None] * offsets[movable]
    nodes, elems, specs = mesh.raw()
    return build_tet_mesh(Y, elems, specs)


def save_mesh(mesh: TetMesh, path) -> None:
    """HODG-MESH v1 with a `dim 3` line: `x y z` nodes, `T a b c d`
    elements, patch faces as node triples (hodg/mesh.py:431-447)."""
    with open(path, "w") as fh:
        fh.write("hodg-mesh 1\ndim 3\n")
        fh.write(f"nodes {mesh.n_nodes}\n")
        for x, y, z in mesh.node_xy:
            fh.write(f"{float(x)!r} {float(y)!r} {float(z)!r}\n")
        fh.write(f"cells {mesh.n_cells}\n")
        for t in mesh.cell_nodes:
            fh.write("T " + " ".join(str(int(v)) for v in t) + "\n")
        fh.write(f"patches {len(mesh.patches)}\n")
        for p in mesh.patches:
            fh.write(f"{p.name} {p.kind} {len(p.face_ids)}\n")
            for f in p.face_ids:
                fh.write(" ".join(str(int(v)) for v in mesh.face_nodes[f]) + "\n")


class HodgMeshReader:
    """Record reader for HODG-MESH v1 files (2D: hodg/mesh.py:450-560, and
    this package's `dim 3` variant): the meaningful lines (blank and '#'
    lines skipped) with their 1-based line numbers, consumed section by
    section.  Every syntax error is a MeshParseError naming the line."""

    def __init__(self, path):
        self.path = path
        with open(path) as fh:
            raw = fh.read().splitlines()
        self.n_lines = len(raw)
        self.records = [(i + 1, t.split()) for i, t in enumerate(s.strip() for s in raw)
                        if t and not t.startswith("#")]
        self.pos = 0

    def fail(self, line_no, msg):
        return MeshParseError(self.path, line_no, msg)

    def take(self, what):
        """The next record, or an error at the end of the file."""
        if self.pos >= len(self.records):
            raise self.fail(self.n_lines, f"expected {what}")
        rec = self.records[self.pos]
        self.pos += 1
        return rec

    def at_end(self) -> bool:
        return self.pos >= len(self.records)

    def expect(self, words, msg):
        ln, f = self.take(msg)
        if f != list(words):
            raise self.fail(ln, msg)

    def count(self, word) -> int:
        ln, f = self.take(f"'{word} N'")
        if len(f) != 2 or f[0] != word:
            raise self.fail(ln, f"expected '{word} N'")
        try:
            return int(f[1])
        except ValueError:
            raise self.fail(ln, f"bad {word} count") from None

    def table(self, n, parse, what):
        """n records through parse(fields) -> row; ValueError -> error."""
        rows = []
        for _ in range(n):
            ln, f = self.take(what)
            try:
                rows.append(parse(f))
            except (ValueError, KeyError):
                raise self.fail(ln, f"expected {what}") from None
        return rows

    def patches(self, arity, kinds, optional=False):
        """[(name, kind, [node tuples])]: a 'patches P' section of P
        'name kind count' headers, each followed by `count` faces of `arity`
        node ids."""
        if optional and self.at_end():
            return []
        specs = []
        for _ in range(self.count("patches")):
            ln, f = self.take("'name kind count'")
            if len(f) != 3 or f[1] not in kinds:
                raise self.fail(ln, "expected 'name kind count' with a known kind")
            try:
                n = int(f[2])
            except ValueError:
                raise self.fail(ln, "bad face count") from None
            specs.append((f[0], f[1], self.table(n, lambda g: _ints(g, arity), f"{arity} node ids")))
        return specs


def _ints(fields, n):
    if len(fields) != n:
        raise ValueError
    return tuple(int(v) for v in fields)


def _floats(fields, n):
    if len(fields) != n:
        raise ValueError
    return tuple(float(v) for v in fields)


def load_mesh(path) -> TetMesh:
    """Read a 3D HODG-MESH file; MeshParseError carries the line number
    (hodg/mesh.py:450-560)."""
    rd = HodgMeshReader(path)
    rd.expect(["hodg-mesh", "1"], "expected header 'hodg-mesh 1'")
    rd.expect(["dim", "3"], "expected 'dim 3'")
    X = np.array(rd.table(rd.count("nodes"), lambda f: _floats(f, 3), "'x y z'"), dtype=np.float64).reshape(-1, 3)

    def tet(f):
        if f[0] != "T":
            raise ValueError
        return _ints(f[1:], 4)

    T = np.array(rd.table(rd.count("cells"), tet, "'T a b c d'"), dtype=np.int64).reshape(-1, 4)
    specs = rd.patches(3, BC_KINDS)
    mesh = build_tet_mesh(X, T, specs)
    problems = validate(mesh)
    if problems:
        raise TopologyError(f"{path}: " + "; ".join(problems[:5]))
    return mesh


def validate(mesh: TetMesh) -> list[str]:
    """Invariant checks; violations are returned, not raised
    (hodg/mesh.py:566-629): geometric closure sum(sgn n A) = 0 per element,
    unit normals, face <-> element back references, patch coverage."""
    problems = []
    n_vec = mesh.face_normal[mesh.cell_faces] * (mesh.face_length[mesh.cell_faces] *
                                                  mesh.cell_fsign)[..., None]
    closure = np.linalg.norm(n_vec.sum(axis=1), axis=1)
    scale = mesh.face_length[mesh.cell_faces].sum(axis=1)
    bad = np.flatnonzero(closure > 1e-12 * scale)
    problems += [f"cell {c}: geometric closure violated" for c in bad[:5]]
    nrm = np.linalg.norm(mesh.face_normal, axis=1)
    problems += [f"face {f}: normal not unit length" for f in np.flatnonzero(np.abs(nrm - 1.0) > 1e-14)[:5]]
    fc = mesh.face_cells[mesh.cell_faces]
    me = np.arange(mesh.n_cells)[:, None]
    ok = (fc[..., 0] == me) | (fc[..., 1] == me)
    problems += [f"cell {c}: face does not reference it back" for c in np.flatnonzero(~ok.all(axis=1))[:5]]
    unpatched = (mesh.face_cells[:, 1] < 0) & (mesh.face_patch < 0)
    problems += [f"face {f}: boundary face without a patch" for f in np.flatnonzero(unpatched)[:5]]
    return problems
