"""The reference's own 2D problem on the B200.

The reference solves 2D triangles / bilinear quadrilaterals with 4
variables (`hodg/mesh.py`, `hodg/geometry.py`).  Bilinear quads are not
affine, so the tetrahedral kernels' reference-element trick does not apply;
this module keeps the reference's table-driven discretisation instead --
host setup restated from `hodg/mesh.py:177-425`, `hodg/geometry.py:98-220`,
`hodg/basis.py:40-69`, `hodg/flows.py:23-57` and `hodg/dg.py:549-569` with the
same numpy expressions (tables are bitwise the reference's) -- and runs the
passes with the `hodg2d_*` kernels of libhodg_b200 (csrc/hodg_2d.cu), whose
argument lists are the reference kernels'.  `run2d` is the reference's
iteration loop (`hodg/timestepping.py:256-357`) with the state resident on
the device; it reproduces fixtures/residuals_{dp,mp}.csv
(tests/test_gpu_2d.py).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .physics import AdmissibilityError
from .precision import PrecisionController, PrecisionSchedule
from .quadrature import gauss_legendre_1d, triangle_rule

__all__ = ["Mesh2D", "build_mesh_2d", "generate_quad_grid", "generate_tri_grid", "perturb_interior_nodes",
           "save_mesh_2d", "load_mesh_2d", "write_vtk_2d",
           "compute_geometry_2d", "Device2D", "RunConfig2D", "run2d", "residual_csv_text"]

BC_KINDS = ("far_field", "slip_wall", "no_slip_wall")
_EDGES = {3: ((0, 1), (1, 2), (2, 0)), 4: ((0, 1), (1, 2), (2, 3), (3, 0))}
_EXP2 = np.array([(0, 0), (1, 0), (0, 1), (2, 0), (1, 1), (0, 2)], dtype=np.int64)  # hodg/basis.py:21
_NB2 = {0: 1, 1: 3, 2: 6}


@dataclass
class Patch2D:
    name: str
    kind: str
    face_ids: np.ndarray


@dataclass
class Mesh2D:
    node_xy: np.ndarray
    cell_nodes: np.ndarray
    cell_nvert: np.ndarray
    cell_faces: np.ndarray
    cell_fsign: np.ndarray
    cell_centroid: np.ndarray
    cell_area: np.ndarray
    cell_h: np.ndarray
    face_nodes: np.ndarray
    face_cells: np.ndarray
    face_normal: np.ndarray
    face_length: np.ndarray
    face_patch: np.ndarray
    patches: list = field(default_factory=list)

    @property
    def n_cells(self):
        return self.cell_nodes.shape[0]

    @property
    def n_faces(self):
        return self.face_nodes.shape[0]

    def boundary_kind_codes(self):
        codes = np.zeros(self.n_faces, dtype=np.int8)
        codes[self.face_cells[:, 1] < 0] = -1
        for p, patch in enumerate(self.patches):
            codes[self.face_patch == p] = BC_KINDS.index(patch.kind) + 1
        return codes


def _area_centroid(xy):
    x, y = xy[:, 0], xy[:, 1]
    xn, yn = np.roll(x, -1), np.roll(y, -1)
    cr = x * yn - xn * y
    a = 0.5 * np.sum(cr)
    return float(a), np.array([np.sum((x + xn) * cr) / (6.0 * a), np.sum((y + yn) * cr) / (6.0 * a)])


def build_mesh_2d(node_xy, cells, patch_specs=None) -> Mesh2D:
    node_xy = np.ascontiguousarray(node_xy, dtype=np.float64)
    n = len(cells)
    cn = np.full((n, 4), -1, dtype=np.int32)
    nv = np.zeros(n, dtype=np.int8)
    for c, nodes in enumerate(cells):
        cn[c, : len(nodes)] = nodes
        nv[c] = len(nodes)
    area, cen = np.empty(n), np.empty((n, 2))
    for c in range(n):
        area[c], cen[c] = _area_centroid(node_xy[cn[c, : nv[c]]])
        if area[c] <= 0.0:
            raise ValueError(f"cell {c}: non-positive signed area")
    keys, fnodes, fcells = {}, [], []
    cf = np.full((n, 4), -1, dtype=np.int32)
    cs = np.zeros((n, 4), dtype=np.int8)
    for c in range(n):
        for slot, (ea, eb) in enumerate(_EDGES[int(nv[c])]):
            a, b = int(cn[c, ea]), int(cn[c, eb])
            k = (a, b) if a < b else (b, a)
            fid = keys.get(k)
            if fid is None:
                fid = keys[k] = len(fnodes)
                fnodes.append((a, b))
                fcells.append([c, -1])
                cs[c, slot] = 1
            else:
                fcells[fid][1] = c
                cs[c, slot] = -1
            cf[c, slot] = fid
    fn = np.array(fnodes, dtype=np.int32)
    fc = np.array(fcells, dtype=np.int32)
    d = node_xy[fn[:, 1]] - node_xy[fn[:, 0]]
    ln = np.hypot(d[:, 0], d[:, 1])
    nrm = np.column_stack([d[:, 1], -d[:, 0]]) / ln[:, None]
    fp = np.full(len(fnodes), -1, dtype=np.int32)
    patches = []
    for p, (name, kind, pairs) in enumerate(patch_specs or []):
        ids = [keys[(min(a, b), max(a, b))] for a, b in pairs]
        fp[ids] = p
        patches.append(Patch2D(name, kind, np.array(sorted(ids), dtype=np.int32)))
    return Mesh2D(node_xy, cn, nv, cf, cs, cen, area, np.sqrt(area), fn, fc, nrm, ln, fp, patches)


def _grid_nodes(nx, ny, extent):
    x0, y0, x1, y1 = extent
    X, Y = np.meshgrid(np.linspace(x0, x1, nx + 1), np.linspace(y0, y1, ny + 1), indexing="xy")
    return np.column_stack([X.ravel(), Y.ravel()])


def _sides(nx, ny, bc):
    bc = {s: bc for s in ("bottom", "right", "top", "left")} if isinstance(bc, str) else bc

    def nid(i, j):
        return j * (nx + 1) + i

    return [("bottom", bc["bottom"], [(nid(i, 0), nid(i + 1, 0)) for i in range(nx)]),
            ("right", bc["right"], [(nid(nx, j), nid(nx, j + 1)) for j in range(ny)]),
            ("top", bc["top"], [(nid(i + 1, ny), nid(i, ny)) for i in range(nx)]),
            ("left", bc["left"], [(nid(0, j + 1), nid(0, j)) for j in range(ny)])]


def generate_quad_grid(nx, ny, extent=(0.0, 0.0, 1.0, 1.0), bc="far_field") -> Mesh2D:
    """hodg/mesh.py:361-376."""
    cells = [(j * (nx + 1) + i, j * (nx + 1) + i + 1, (j + 1) * (nx + 1) + i + 1, (j + 1) * (nx + 1) + i)
             for j in range(ny) for i in range(nx)]
    return build_mesh_2d(_grid_nodes(nx, ny, extent), cells, _sides(nx, ny, bc))


def generate_tri_grid(nx, ny, extent=(0.0, 0.0, 1.0, 1.0), bc="far_field") -> Mesh2D:
    """hodg/mesh.py:379-393."""
    cells = []
    for j in range(ny):
        for i in range(nx):
            a, b = j * (nx + 1) + i, j * (nx + 1) + i + 1
            c, d = (j + 1) * (nx + 1) + i + 1, (j + 1) * (nx + 1) + i
            cells += [(a, b, c), (a, c, d)]
    return build_mesh_2d(_grid_nodes(nx, ny, extent), cells, _sides(nx, ny, bc))


def perturb_interior_nodes(m: Mesh2D, amplitude, seed=0) -> Mesh2D:
    """hodg/mesh.py:396-425."""
    rng = np.random.default_rng(seed)
    bnodes = set(m.face_nodes[m.face_cells[:, 1] < 0].ravel().tolist())
    short = np.full(m.node_xy.shape[0], np.inf)
    for f in range(m.n_faces):
        a, b = m.face_nodes[f]
        short[a] = min(short[a], m.face_length[f])
        short[b] = min(short[b], m.face_length[f])
    xy = m.node_xy.copy()
    off = rng.uniform(-1.0, 1.0, size=xy.shape)
    for i in range(xy.shape[0]):
        if i not in bnodes:
            xy[i] += amplitude * short[i] * off[i]
    cells = [tuple(m.cell_nodes[c, : m.cell_nvert[c]]) for c in range(m.n_cells)]
    specs = [(p.name, p.kind, [tuple(m.face_nodes[f]) for f in p.face_ids]) for p in m.patches]
    return build_mesh_2d(xy, cells, specs)


# ---------------------------------------------------------------------------
# HODG-MESH v1 (hodg/mesh.py:431-560): the reference's 2D plain-text format


def _mesh_2d_records(m: Mesh2D):
    """The HODG-MESH v1 lines of a 2D mesh, section by section."""
    yield "hodg-mesh 1"
    yield f"nodes {m.node_xy.shape[0]}"
    yield from (f"{float(x)!r} {float(y)!r}" for x, y in m.node_xy)
    yield f"cells {m.n_cells}"
    tag = {3: "t", 4: "q"}
    for nodes, nv in zip(m.cell_nodes, m.cell_nvert):
        yield " ".join([tag[int(nv)]] + [str(int(k)) for k in nodes[: int(nv)]])
    yield f"patches {len(m.patches)}"
    for p in m.patches:
        yield f"{p.name} {p.kind} {len(p.face_ids)}"
        yield from (f"{int(a)} {int(b)}" for a, b in m.face_nodes[p.face_ids])


def save_mesh_2d(m: Mesh2D, path) -> None:
    """The reference's 2D HODG-MESH v1 writer (hodg/mesh.py:431-447):
    byte-identical output (floats by repr)."""
    with open(path, "w") as fh:
        fh.write("\n".join(_mesh_2d_records(m)) + "\n")


def load_mesh_2d(path) -> Mesh2D:
    """Read the reference's 2D HODG-MESH v1 (hodg/mesh.py:450-560):
    MeshParseError with the line number on malformed input, TopologyError on
    bad connectivity.  Cells are 't i j k' or 'q i j k l'; the patch section
    is optional."""
    from .mesh import HodgMeshReader, TopologyError

    rd = HodgMeshReader(path)
    rd.expect(["hodg-mesh", "1"], "expected header 'hodg-mesh 1'")
    nodes = rd.table(rd.count("nodes"), lambda f: tuple(float(v) for v in _arity(f, 2)), "'x y'")
    xy = np.array(nodes, dtype=np.float64).reshape(-1, 2)
    arity = {"t": 3, "q": 4}
    cells = rd.table(rd.count("cells"), lambda f: tuple(int(v) for v in _arity(f[1:], arity[f[0]])),
                     "'t i j k' or 'q i j k l'")
    specs = rd.patches(2, BC_KINDS, optional=True)
    try:
        return build_mesh_2d(xy, cells, specs)
    except (ValueError, KeyError) as e:
        raise TopologyError(f"{path}: {e}") from None


def _arity(fields, n):
    if len(fields) != n:
        raise ValueError
    return fields


def write_vtk_2d(path, m: Mesh2D, t: "Tables2D", coeffs, gamma: float = 1.4) -> None:
    """Cell-mean flow field (rho, u, v, p, Mach) of a state -- a device
    tensor or an array -- on the unstructured grid, in the reference's
    legacy-VTK layout (hodg/output.py:54-83; byte-identical for the same
    state).  The means are the reference's einsum (hodg/dg.py:666-668)."""
    if hasattr(coeffs, "detach"):
        coeffs = coeffs.detach().cpu().numpy()
    means = np.einsum("cvj,cj->cv", np.asarray(coeffs).astype(np.float64), t.basis_mean)
    rho = means[:, 0]
    u = means[:, 1] / rho
    v = means[:, 2] / rho
    p = (gamma - 1.0) * (means[:, 3] - 0.5 * rho * (u * u + v * v))
    a = np.sqrt(np.maximum(gamma * p / rho, 0.0))
    mach = np.divide(np.hypot(u, v), a, out=np.zeros_like(a), where=a > 0)
    with open(path, "w") as fh:
        fh.write("# vtk DataFile Version 3.0\n")
        fh.write("hodg cell-mean flow field\n")
        fh.write("ASCII\nDATASET UNSTRUCTURED_GRID\n")
        fh.write(f"POINTS {m.node_xy.shape[0]} double\n")
        for x, y in m.node_xy:
            fh.write(f"{float(x)!r} {float(y)!r} 0.0\n")
        sizes = m.cell_nvert.astype(np.int64)
        fh.write(f"CELLS {m.n_cells} {int(np.sum(sizes + 1))}\n")
        for c in range(m.n_cells):
            nv = int(sizes[c])
            fh.write(f"{nv} " + " ".join(str(int(n)) for n in m.cell_nodes[c, :nv]) + "\n")
        fh.write(f"CELL_TYPES {m.n_cells}\n")
        for c in range(m.n_cells):
            fh.write("5\n" if sizes[c] == 3 else "9\n")
        fh.write(f"CELL_DATA {m.n_cells}\n")
        for name, vals in (("rho", rho), ("u", u), ("v", v), ("p", p), ("Mach", mach)):
            fh.write(f"SCALARS {name} double 1\nLOOKUP_TABLE default\n")
            for val in vals:
                fh.write(f"{float(val)!r}\n")


# ---------------------------------------------------------------------------
# geometry tables (hodg/geometry.py:120-220)


@dataclass
class Tables2D:
    order: int
    nb: int
    vol_xy: np.ndarray
    vol_w: np.ndarray
    vol_basis: np.ndarray
    vol_gx: np.ndarray
    vol_gy: np.ndarray
    face_w: np.ndarray
    fbl: np.ndarray
    fbr: np.ndarray
    minv: np.ndarray
    basis_mean: np.ndarray


def _basis(x, y, xc, yc, h, nb):
    X = (x - xc) / h
    Y = (y - yc) / h
    out = np.empty(X.shape + (nb,))
    for j in range(nb):
        px, py = _EXP2[j]
        out[..., j] = X ** px * Y ** py
    return out


def _grads(x, y, xc, yc, h, nb):
    X = (x - xc) / h
    Y = (y - yc) / h
    gx = np.zeros(X.shape + (nb,))
    gy = np.zeros(X.shape + (nb,))
    for j in range(nb):
        px, py = _EXP2[j]
        if px > 0:
            gx[..., j] = px * X ** (px - 1) * Y ** py / h
        if py > 0:
            gy[..., j] = py * X ** px * Y ** (py - 1) / h
    return gx, gy


def _quad_map(corners, ref):
    xi, eta = ref[:, 0], ref[:, 1]
    shape = 0.25 * np.column_stack([(1 - xi) * (1 - eta), (1 + xi) * (1 - eta), (1 + xi) * (1 + eta),
                                    (1 - xi) * (1 + eta)])
    dxi = 0.25 * np.column_stack([-(1 - eta), (1 - eta), (1 + eta), -(1 + eta)])
    deta = 0.25 * np.column_stack([-(1 - xi), -(1 + xi), (1 + xi), (1 - xi)])
    xy = shape @ corners
    jx = dxi @ corners
    jy = deta @ corners
    return xy, jx[:, 0] * jy[:, 1] - jx[:, 1] * jy[:, 0]


def compute_geometry_2d(m: Mesh2D, order: int) -> Tables2D:
    nb = _NB2[order]
    n = m.n_cells
    tb, tw = triangle_rule(max(2 * order, 1))
    g1, gw = gauss_legendre_1d(order + 1)
    XI, ETA = np.meshgrid(g1, g1, indexing="ij")
    qp = np.column_stack([XI.ravel(), ETA.ravel()])
    qw = np.outer(gw, gw).ravel()
    nqv = max(tw.size if np.any(m.cell_nvert == 3) else 0, qw.size if np.any(m.cell_nvert == 4) else 0)
    vxy = np.zeros((n, nqv, 2))
    vw = np.zeros((n, nqv))
    vb = np.zeros((n, nqv, nb))
    vgx = np.zeros((n, nqv, nb))
    vgy = np.zeros((n, nqv, nb))
    minv = np.zeros((n, nb, nb))
    bmean = np.zeros((n, nb))
    for c in range(n):
        nv = int(m.cell_nvert[c])
        corners = m.node_xy[m.cell_nodes[c, :nv]]
        if nv == 3:
            xy = tb @ corners
            w = tw * m.cell_area[c]
        else:
            xy, det = _quad_map(corners, qp)
            w = qw * det
        k = xy.shape[0]
        xc, yc = m.cell_centroid[c]
        h = m.cell_h[c]
        b = _basis(xy[:, 0], xy[:, 1], xc, yc, h, nb)
        gx, gy = _grads(xy[:, 0], xy[:, 1], xc, yc, h, nb)
        vxy[c, :k], vw[c, :k], vb[c, :k], vgx[c, :k], vgy[c, :k] = xy, w, b, gx, gy
        minv[c] = np.linalg.inv(np.einsum("q,qj,qk->jk", w, b, b))
        bmean[c] = (w @ b) / m.cell_area[c]
    nqf = order + 1
    t1, w1 = gauss_legendre_1d(nqf)
    fxy = np.zeros((m.n_faces, nqf, 2))
    fw = np.zeros((m.n_faces, nqf))
    a_xy = m.node_xy[m.face_nodes[:, 0]]
    b_xy = m.node_xy[m.face_nodes[:, 1]]
    for q in range(nqf):
        s = 0.5 * (1.0 + t1[q])
        fxy[:, q, :] = a_xy + s * (b_xy - a_xy)
        fw[:, q] = 0.5 * w1[q] * m.face_length
    fbl = np.zeros((m.n_faces, nqf, nb))
    fbr = np.zeros((m.n_faces, nqf, nb))
    for f in range(m.n_faces):
        for side, cell in enumerate(m.face_cells[f]):
            if cell < 0:
                continue
            xc, yc = m.cell_centroid[cell]
            vals = _basis(fxy[f, :, 0], fxy[f, :, 1], xc, yc, m.cell_h[cell], nb)
            (fbl if side == 0 else fbr)[f] = vals
    return Tables2D(order, nb, vxy, vw, vb, vgx, vgy, fw, fbl, fbr, minv, bmean)


# ---------------------------------------------------------------------------
# flows / projection (hodg/flows.py:23-57, hodg/dg.py:549-569)


def freestream_2d(gamma, R, mach, angle_deg):
    a = np.sqrt(gamma * R * 1.0)
    ang = np.deg2rad(angle_deg)
    u, v, p = mach * a * np.cos(ang), mach * a * np.sin(ang), 1.0 * R * 1.0
    e = p / (gamma - 1.0) + 0.5 * 1.0 * (u * u + v * v)
    return (1.0, u, v, p), np.array([1.0, 1.0 * u, 1.0 * v, e])


def vortex_2d(gamma, R, mach, angle_deg, beta, x0, y0, x, y):
    (_, ui, vi, _), _ = freestream_2d(gamma, R, mach, angle_deg)
    xr = np.asarray(x, dtype=np.float64) - x0 - ui * 0.0
    yr = np.asarray(y, dtype=np.float64) - y0 - vi * 0.0
    r2 = xr * xr + yr * yr
    env = np.exp(0.5 * (1.0 - r2))
    vs = np.sqrt(R)
    u = ui - beta / (2.0 * np.pi) * yr * env * vs
    v = vi + beta / (2.0 * np.pi) * xr * env * vs
    T = 1.0 - (gamma - 1.0) * beta * beta / (8.0 * gamma * np.pi * np.pi) * np.exp(1.0 - r2)
    rho = T ** (1.0 / (gamma - 1.0))
    return rho, u, v, rho * R * T


def pulse_2d(gamma, R, amplitude, sigma, x0, y0, x, y, mach=0.0, angle_deg=0.0):
    """hodg/flows.py:60-73."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    r2 = (x - x0) ** 2 + (y - y0) ** 2
    p = R * (1.0 + amplitude * np.exp(-0.5 * r2 / (sigma * sigma)))
    rho = (p / R) ** (1.0 / gamma)
    if mach > 0.0:
        (_, ui, vi, _), _ = freestream_2d(gamma, R, mach, angle_deg)
        u, v = np.full_like(p, ui), np.full_like(p, vi)
    else:
        u, v = np.zeros_like(p), np.zeros_like(p)
    return rho, u, v, p


def project_2d(m: Mesh2D, t: Tables2D, prim, gamma):
    x = t.vol_xy[:, :, 0].ravel()
    rho, u, v, p = (np.broadcast_to(np.asarray(a, dtype=np.float64), x.shape) for a in prim)
    if np.any(rho <= 0.0) or np.any(p <= 0.0):
        raise AdmissibilityError("initial field is inadmissible")
    e = p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v)
    q = np.stack([rho, rho * u, rho * v, e], axis=-1).reshape(m.n_cells, t.vol_w.shape[1], 4)
    proj = np.einsum("cq,cqj,cqv->cvj", t.vol_w, t.vol_basis, q)
    return np.ascontiguousarray(np.einsum("cjk,cvk->cvj", t.minv, proj))


# ---------------------------------------------------------------------------
# device passes


class Device2D:
    """Tables uploaded once per precision; passes over device arrays."""

    def __init__(self, m: Mesh2D, t: Tables2D, gamma, qinf, flux_kind=0, mu=0.0, device="cuda", R=1.0, Pr=0.72,
                 ivis=0):
        import torch

        self.L = _lib.lib()
        self.m, self.t, self.gamma, self.mu, self.flux_kind = m, t, float(gamma), float(mu), flux_kind
        self.R, self.Pr, self.ivis = float(R), float(Pr), int(ivis)
        if self.ivis not in (0, 1):
            raise ValueError("ivis must be 0 or 1")
        if self.ivis and flux_kind != 0:
            raise ValueError("the viscous passes use the Roe flux, as the reference's")
        self.dev = torch.device(device)
        self.qinf = np.asarray(qinf, dtype=np.float64)
        bc = m.boundary_kind_codes()
        if np.any(bc < 0):
            raise ValueError("boundary face without a patch")

        def up(a, dt=None):
            a = np.ascontiguousarray(a if dt is None else a.astype(dt))
            return torch.from_numpy(a).to(self.dev)

        self.face_cells = up(m.face_cells.astype(np.int32))
        self.bc = up(bc)
        self.cell_nv = up(m.cell_nvert.astype(np.int8))
        self.cell_faces = up(m.cell_faces.astype(np.int32))
        self.cell_fsign = up(m.cell_fsign.astype(np.int8))
        self.minv = up(t.minv)
        self.bmean = up(t.basis_mean)
        self.h = up(m.cell_h)
        self._tabs = {}
        self._up = up
        self.errf = torch.zeros(m.n_faces, dtype=torch.uint8, device=self.dev)
        self.errc = torch.zeros(m.n_cells, dtype=torch.uint8, device=self.dev)

    def tabs(self, prec):
        d = self._tabs.get(prec)
        if d is None:
            dt = np.float64 if prec == _lib.PREC_F64 else np.float32
            up = self._up
            t, m = self.t, self.m
            d = dict(fbL=up(t.fbl, dt), fbR=up(t.fbr, dt), fnx=up(m.face_normal[:, 0], dt),
                     fny=up(m.face_normal[:, 1], dt), qinf=up(self.qinf, dt), vol_w=up(t.vol_w, dt),
                     vol_b=up(t.vol_basis, dt), vol_gx=up(t.vol_gx, dt), vol_gy=up(t.vol_gy, dt), face_w=up(t.face_w, dt),
                     minv=up(t.minv, dt))
            self._tabs[prec] = d
        return d

    def _raise(self, err, msg, key, iteration):
        if bool(err.any()):
            idx = int(err.nonzero()[0, 0])
            raise AdmissibilityError(msg, iteration=iteration, **{key: idx})

    def _prec(self, coeffs):
        import torch

        return _lib.PREC_F64 if coeffs.dtype == torch.float64 else _lib.PREC_MIXED

    def aux_gradient(self, coeffs, iteration=None):
        """compute_aux_gradient (hodg/dg.py:572-591): qhat_pass + aux_pass;
        returns z as (n_cells, 2, 4, nb) at the state precision."""
        import torch

        prec = self._prec(coeffs)
        d = self.tabs(prec)
        m, t = self.m, self.t
        nqf = t.face_w.shape[1]
        P, s = _lib.ptr, _lib.stream_ptr()
        qhat = torch.zeros((m.n_faces, nqf, 4), dtype=coeffs.dtype, device=self.dev)
        self.errf.zero_()
        _lib.check(self.L.hodg2d_qhat_pass(prec, m.n_faces, nqf, t.nb, P(coeffs), P(d["fbL"]), P(d["fbR"]),
                                           P(self.face_cells), P(self.bc), P(d["fnx"]), P(d["fny"]), P(d["qinf"]),
                                           self.gamma, P(qhat), P(self.errf), s), "hodg2d_qhat_pass")
        self._raise(self.errf, "inadmissible face trace", "face", iteration)
        aux = torch.empty((m.n_cells, 2, 4, t.nb), dtype=coeffs.dtype, device=self.dev)
        _lib.check(self.L.hodg2d_aux_pass(prec, m.n_cells, t.nb, t.vol_w.shape[1], nqf, 4, P(coeffs), P(qhat),
                                          P(d["vol_w"]), P(d["vol_b"]), P(d["vol_gx"]), P(d["vol_gy"]),
                                          P(self.cell_nv), P(self.cell_faces), P(self.cell_fsign), P(d["face_w"]),
                                          P(d["fbL"]), P(d["fbR"]), P(d["fnx"]), P(d["fny"]), P(d["minv"]), P(aux),
                                          s), "hodg2d_aux_pass")
        return aux

    def face_flux_ns(self, coeffs, aux, iteration=None):
        """face_flux_pass with ivis = 1 (hodg/dg.py:594-621): (finv, fvis, fqhat)."""
        import torch

        prec = self._prec(coeffs)
        d = self.tabs(prec)
        m, t = self.m, self.t
        nqf = t.face_w.shape[1]
        P, s = _lib.ptr, _lib.stream_ptr()
        finv, fvis, fqhat = (torch.zeros((m.n_faces, nqf, 4), dtype=coeffs.dtype, device=self.dev) for _ in range(3))
        self.errf.zero_()
        _lib.check(self.L.hodg2d_flux_pass_ns(prec, m.n_faces, nqf, t.nb, P(coeffs), P(aux), P(d["fbL"]),
                                              P(d["fbR"]), P(self.face_cells), P(self.bc), P(d["fnx"]), P(d["fny"]),
                                              P(d["qinf"]), self.gamma, self.R, self.mu, self.Pr, P(finv), P(fvis),
                                              P(fqhat), P(self.errf), s), "hodg2d_flux_pass_ns")
        self._raise(self.errf, "inadmissible face trace", "face", iteration)
        return finv, fvis, fqhat

    def accumulate_ns(self, coeffs, aux, finv, fvis, iteration=None):
        """accumulate_rhs with ivis = 1 (hodg/dg.py:624-649); float64 residual."""
        import torch

        prec = self._prec(coeffs)
        d = self.tabs(prec)
        m, t = self.m, self.t
        P, s = _lib.ptr, _lib.stream_ptr()
        res = torch.empty((m.n_cells, 4, t.nb), dtype=torch.float64, device=self.dev)
        self.errc.zero_()
        _lib.check(self.L.hodg2d_rhs_pass_ns(prec, m.n_cells, t.nb, t.vol_w.shape[1], t.face_w.shape[1], 4,
                                             P(coeffs), P(aux), P(finv), P(fvis), P(d["vol_w"]), P(d["vol_b"]),
                                             P(d["vol_gx"]), P(d["vol_gy"]), P(self.cell_nv), P(self.cell_faces),
                                             P(self.cell_fsign), P(d["face_w"]), P(d["fbL"]), P(d["fbR"]),
                                             P(self.minv), self.gamma, self.R, self.mu, self.Pr, P(res), P(self.errc),
                                             s), "hodg2d_rhs_pass_ns")
        self._raise(self.errc, "inadmissible volume state", "cell", iteration)
        return res

    def rhs(self, coeffs, iteration=None):
        """aux gradient (viscous runs only), flux_pass, rhs_pass
        (hodg/dg.py:652-663); float64 residual."""
        import torch

        if self.ivis:
            aux = self.aux_gradient(coeffs, iteration)
            finv, fvis, _ = self.face_flux_ns(coeffs, aux, iteration)
            return self.accumulate_ns(coeffs, aux, finv, fvis, iteration)
        prec = self._prec(coeffs)
        d = self.tabs(prec)
        m, t = self.m, self.t
        nqf = t.face_w.shape[1]
        finv = torch.zeros((m.n_faces, nqf, 4), dtype=coeffs.dtype, device=self.dev)
        self.errf.zero_()
        P = _lib.ptr
        s = _lib.stream_ptr()
        _lib.check(self.L.hodg2d_flux_pass(prec, m.n_faces, nqf, t.nb, P(coeffs), P(d["fbL"]), P(d["fbR"]),
                                           P(self.face_cells), P(self.bc), P(d["fnx"]), P(d["fny"]), P(d["qinf"]),
                                           self.gamma, self.flux_kind, P(finv), P(self.errf), s), "hodg2d_flux_pass")
        self._raise(self.errf, "inadmissible face trace", "face", iteration)
        res = torch.empty((m.n_cells, 4, t.nb), dtype=torch.float64, device=self.dev)
        self.errc.zero_()
        _lib.check(self.L.hodg2d_rhs_pass(prec, m.n_cells, t.nb, t.vol_w.shape[1], nqf, 4, P(coeffs), P(finv),
                                          P(d["vol_w"]), P(d["vol_b"]), P(d["vol_gx"]), P(d["vol_gy"]),
                                          P(self.cell_nv), P(self.cell_faces), P(self.cell_fsign), P(d["face_w"]),
                                          P(d["fbL"]), P(d["fbR"]), P(self.minv), self.gamma, P(res), P(self.errc),
                                          s), "hodg2d_rhs_pass")
        self._raise(self.errc, "inadmissible volume state", "cell", iteration)
        return res

    def local_dt(self, coeffs, cfl, order, iteration=None):
        import torch

        prec = _lib.PREC_F64 if coeffs.dtype == torch.float64 else _lib.PREC_MIXED
        out = torch.empty(self.m.n_cells, dtype=torch.float64, device=self.dev)
        self.errc.zero_()
        _lib.check(self.L.hodg2d_dt_pass(prec, self.m.n_cells, self.t.nb, _lib.ptr(coeffs), _lib.ptr(self.bmean),
                                         _lib.ptr(self.h), self.gamma, self.mu, cfl, order, _lib.ptr(out),
                                         _lib.ptr(self.errc), _lib.stream_ptr()), "hodg2d_dt_pass")
        self._raise(self.errc, "inadmissible cell mean", "cell", iteration)
        return out

    def rk2_step(self, u, dtc, iteration=None):
        """hodg/timestepping.py:192-205 on device; returns (new state, first-stage residual)."""
        import torch

        prec = _lib.PREC_F64 if u.dtype == torch.float64 else _lib.PREC_MIXED
        per = u.shape[1] * u.shape[2]
        r0 = self.rhs(u, iteration)
        u1 = torch.empty_like(u)
        _lib.check(self.L.hodg2d_axpy(prec, u.shape[0], per, _lib.ptr(u), _lib.ptr(r0), _lib.ptr(dtc), _lib.ptr(u1),
                                      _lib.stream_ptr()), "hodg2d_axpy")
        r1 = self.rhs(u1, iteration)
        out = torch.empty_like(u)
        _lib.check(self.L.hodg2d_combine(prec, u.shape[0], per, _lib.ptr(u), _lib.ptr(u1), _lib.ptr(r1),
                                         _lib.ptr(dtc), _lib.ptr(out), _lib.stream_ptr()), "hodg2d_combine")
        return out, r0


@dataclass
class RunConfig2D:
    """The reference RunConfig fields its fixture runs use (hodg/config.py:28-75)."""

    mesh_path: str | None = None  # HODG-MESH v1 file instead of the generator
    gen_kind: str = "quad"
    gen_nx: int = 16
    gen_ny: int = 16
    gen_extent: tuple = (0.0, 0.0, 1.0, 1.0)
    gen_bc: object = "far_field"
    gamma: float = 1.4
    R: float = 1.0
    mu_dyn: float | None = None
    Pr: float = 0.72
    ivis: int = 0
    mach: float = 0.3
    angle_deg: float = 0.0
    reynolds: float | None = None
    initial_kind: str = "freestream"  # freestream | vortex | pulse
    vortex_beta: float = 5.0
    initial_x0: float = 0.0
    initial_y0: float = 0.0
    pulse_amplitude: float = 0.2
    pulse_sigma: float = 0.1
    order: int = 1
    cfl: float = 0.3
    dt_mode: str = "local"
    dt_floor: float = 0.0
    dt_fixed: float | None = None
    t_final: float | None = None
    max_iterations: int = 100
    residual_target: float | None = None
    log_every: int = 1
    precision_mode: str = "dp"
    switch_iter: int = 0
    window: int = 200
    factor: float = 2.0
    flux_kind: int = 0

    def mu(self) -> float:
        """hodg/config.py:102-111: explicit mu, else Mach * a / Re for viscous runs."""
        if self.mu_dyn is not None:
            return float(self.mu_dyn)
        if self.ivis and self.reynolds:
            return self.mach * (self.gamma * self.R) ** 0.5 / self.reynolds
        return 0.0


@dataclass
class History2D:
    iterations: list = field(default_factory=list)
    res: list = field(default_factory=list)
    dts: list = field(default_factory=list)
    precision: list = field(default_factory=list)


def run2d(cfg: RunConfig2D):
    """hodg/timestepping.py:256-357 with the passes on the GPU."""
    import torch

    if cfg.mesh_path is not None:
        m = load_mesh_2d(cfg.mesh_path)
    else:
        gen = generate_quad_grid if cfg.gen_kind == "quad" else generate_tri_grid
        m = gen(cfg.gen_nx, cfg.gen_ny, cfg.gen_extent, cfg.gen_bc)
    t = compute_geometry_2d(m, cfg.order)
    prim_inf, qinf = freestream_2d(cfg.gamma, cfg.R, cfg.mach, cfg.angle_deg)
    x = t.vol_xy[:, :, 0].ravel()
    y = t.vol_xy[:, :, 1].ravel()
    if cfg.initial_kind == "vortex":
        prim = vortex_2d(cfg.gamma, cfg.R, cfg.mach, cfg.angle_deg, cfg.vortex_beta, cfg.initial_x0,
                         cfg.initial_y0, x, y)
    elif cfg.initial_kind == "pulse":
        prim = pulse_2d(cfg.gamma, cfg.R, cfg.pulse_amplitude, cfg.pulse_sigma, cfg.initial_x0, cfg.initial_y0, x, y,
                        cfg.mach, cfg.angle_deg)
    else:
        prim = prim_inf
    u = torch.from_numpy(project_2d(m, t, prim, cfg.gamma)).cuda()
    dev = Device2D(m, t, cfg.gamma, qinf, cfg.flux_kind, mu=cfg.mu(), R=cfg.R, Pr=cfg.Pr, ivis=cfg.ivis)
    ctrl = PrecisionController(PrecisionSchedule(cfg.precision_mode, cfg.switch_iter, cfg.window, cfg.factor))
    sched = ctrl.schedule
    if sched.mode in ("sp", "mp_rebound") or (sched.mode == "mp_fixed" and sched.switch_iter > 0):
        u = u.to(torch.float32)
    hist = History2D()
    area = m.cell_area
    t_sim = 0.0
    for it in range(cfg.max_iterations):
        bits, _ = ctrl.decide(it, [r[0] for r in hist.res])
        if bits == 64 and u.dtype == torch.float32:
            u = u.to(torch.float64)
        dts = dev.local_dt(u, cfg.cfl, cfg.order, it)
        if cfg.dt_floor > 0.0:
            dts = torch.clamp_min(dts, cfg.dt_floor)
        if cfg.dt_mode == "global":
            dmin = cfg.dt_fixed if cfg.dt_fixed is not None else float(dts.min().item())
            if cfg.t_final is not None:
                if t_sim >= cfg.t_final - 1e-14:
                    break
                dmin = min(dmin, cfg.t_final - t_sim)
            dtv = torch.full_like(dts, dmin)
        else:
            dmin = float(dts.min().item())
            dtv = dts
        u, r0 = dev.rk2_step(u, dtv, it)
        if cfg.dt_mode == "global":
            t_sim += dmin
        if cfg.log_every and (it % cfg.log_every == 0 or it == cfg.max_iterations - 1):
            r = r0[:, :, 0].cpu().numpy()
            res4 = np.sqrt(np.sum(area[:, None] * r * r, axis=0))  # hodg/timestepping.py:208-211
            if not np.all(np.isfinite(res4)):
                from .timestepping import SolverDivergedError

                raise SolverDivergedError(it, hist)
            hist.iterations.append(it)
            hist.res.append(tuple(float(v) for v in res4))
            hist.dts.append(dmin)
            hist.precision.append(bits)
            if cfg.residual_target is not None and np.all(res4 < cfg.residual_target):
                break
    return u, hist, m, t


def residual_csv_text(hist) -> str:
    """hodg/output.py:17-28."""
    out = ["iter,res_rho,res_rhou,res_rhov,res_e,dt,precision"]
    for it, res, dt, bits in zip(hist.iterations, hist.res, hist.dts, hist.precision):
        out.append(f"{it},{res[0]!r},{res[1]!r},{res[2]!r},{res[3]!r},{dt!r},{bits}")
    return "\n".join(out) + "\n"
