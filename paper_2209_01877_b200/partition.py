"""Mesh partitioning and halo plans for multi-GPU runs.

Not in the reference (single node, `SPEC.md:15`).  METIS-free recursive
coordinate bisection on element centroids: split along the longest axis of
the part's bounding box, ordering by (coordinate, element id) -- integer
tie-break, no floating-point sums -- so the partition map is bit-exact with
its restatement (oracle/partition.py, tests/test_partition.py).

Each rank owns a set of elements and keeps ghost copies of the elements
across its partition faces.  Local numbering: owned elements ascending by
global id, then ghosts ordered by (owner rank, global id), so the rows a
rank receives from one peer are one contiguous block.  Local faces: every
face touching an owned element, interior-of-partition faces first, then the
partition faces; each keeps its global left/right orientation, so the
partition-face flux is computed bit-identically on both ranks and a
partitioned run equals the single-GPU run bitwise (up to the order of the
global residual-norm sum).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .mesh import BoundaryPatch, TetMesh

__all__ = ["rcb_partition", "LocalPart", "build_local", "HaloExchange", "NativeHaloExchange"]


def rcb_partition(points: np.ndarray, nparts: int) -> np.ndarray:
    """Part id per point (int32) by recursive coordinate bisection: the
    library's `hodg_partition_rcb` (host C++, csrc/halo.cu)."""
    from . import _lib

    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    n = pts.shape[0]
    if nparts < 1:
        raise ValueError("nparts must be >= 1")
    if nparts > max(n, 1):
        raise ValueError("more parts than elements")
    parts = np.zeros(n, dtype=np.int32)
    if n:
        _lib.check(_lib.load().hodg_partition_rcb(n, pts.ctypes.data, int(nparts), parts.ctypes.data),
                   "hodg_partition_rcb")
    return parts


@dataclass
class LocalPart:
    rank: int
    nparts: int
    owned: np.ndarray  # global ids, ascending
    ghosts: np.ndarray  # global ids, by (owner, id)
    ghost_owner: np.ndarray
    face_gid: np.ndarray  # global face id of each local face
    n_inner_faces: int
    mesh: TetMesh  # local mesh: owned + ghost elements, local faces
    send_idx: dict = field(default_factory=dict)  # peer -> local (owned) row indices, ascending gid
    recv_range: dict = field(default_factory=dict)  # peer -> (first local row, count)

    @property
    def n_owned(self) -> int:
        return self.owned.size

    @property
    def n_rows(self) -> int:
        return self.owned.size + self.ghosts.size

    @property
    def n_faces(self) -> int:
        return self.face_gid.size


def build_local(mesh: TetMesh, parts: np.ndarray, rank: int) -> LocalPart:
    """The rank's local problem and its halo plan."""
    nparts = int(parts.max()) + 1
    owned = np.flatnonzero(parts == rank).astype(np.int64)
    mine = parts == rank
    fc = mesh.face_cells.astype(np.int64)
    l_own = mine[fc[:, 0]]
    r_exists = fc[:, 1] >= 0
    r_own = np.where(r_exists, mine[np.maximum(fc[:, 1], 0)], False)
    touch = l_own | r_own
    cross = touch & r_exists & (l_own != r_own)
    inner_f = np.flatnonzero(touch & ~cross)
    cross_f = np.flatnonzero(cross)
    face_gid = np.concatenate([inner_f, cross_f])
    # ghosts: the non-owned side of partition faces, by (owner, gid)
    other = np.where(l_own[cross_f], fc[cross_f, 1], fc[cross_f, 0])
    g = np.unique(other)
    g = g[np.lexsort((g, parts[g]))]
    local = np.full(mesh.n_cells, -1, dtype=np.int64)
    local[owned] = np.arange(owned.size)
    local[g] = owned.size + np.arange(g.size)
    elems = np.concatenate([owned, g])
    fmap = np.full(mesh.n_faces, -1, dtype=np.int64)
    fmap[face_gid] = np.arange(face_gid.size)

    lfc = fc[face_gid]
    lfc = np.stack([local[lfc[:, 0]], np.where(lfc[:, 1] >= 0, local[np.maximum(lfc[:, 1], 0)], -1)], axis=1)
    cf = mesh.cell_faces[elems].astype(np.int64)
    lcf = np.where(cf >= 0, fmap[np.maximum(cf, 0)], -1)
    lcf[owned.size:] = -1  # ghosts never gather
    cn = mesh.cell_neighbors[elems].astype(np.int64)
    lcn = np.where(cn >= 0, local[np.maximum(cn, 0)], -1)
    patches = []
    for p in mesh.patches:
        ids = fmap[p.face_ids]
        patches.append(BoundaryPatch(p.name, p.kind, np.sort(ids[ids >= 0]).astype(np.int32)))
    lm = TetMesh(mesh.node_xy, mesh.cell_nodes[elems], lcf.astype(np.int32), mesh.cell_fsign[elems],
                 lcn.astype(np.int32), mesh.cell_centroid[elems], mesh.cell_area[elems], mesh.cell_h[elems],
                 mesh.face_nodes[face_gid], lfc.astype(np.int32), mesh.face_slots[face_gid],
                 mesh.face_normal[face_gid], mesh.face_length[face_gid], mesh.face_patch[face_gid], patches)
    part = LocalPart(rank, nparts, owned, g, parts[g].astype(np.int32), face_gid, int(inner_f.size), lm)
    # receive blocks
    for q in range(nparts):
        sel = np.flatnonzero(part.ghost_owner == q)
        if sel.size:
            part.recv_range[q] = (owned.size + int(sel[0]), int(sel.size))
    # send lists: my owned elements adjacent to each peer's elements, ascending gid
    for q in range(nparts):
        if q == rank:
            continue
        theirs = parts == q
        a = (l_own & r_exists) & np.where(r_exists, theirs[np.maximum(fc[:, 1], 0)], False)
        b = r_own & theirs[fc[:, 0]]
        src = np.unique(np.concatenate([fc[a, 0], fc[b, 1]]))
        if src.size:
            part.send_idx[q] = local[src]
    return part


class HaloExchange:
    """Ghost-row exchange over torch.distributed point-to-point ops: NCCL
    over NVLink on GPUs, gloo on CPU (tests).  `start` packs the send rows
    and posts every receive straight into the ghost block of `rows`, then
    every send; `wait` completes them (on NCCL the current stream waits)."""

    def __init__(self, part: LocalPart, device, group=None):
        import torch

        self.part = part
        self.group = group
        self.device = device
        self.idx = {q: torch.as_tensor(ix, dtype=torch.int64, device=device) for q, ix in part.send_idx.items()}
        self._bufs = {}
        self._work = []

    def start(self, rows):
        import torch
        import torch.distributed as dist

        self._work = []
        for q, (r0, cnt) in sorted(self.part.recv_range.items()):
            self._work.append(dist.irecv(rows[r0:r0 + cnt], src=q, group=self.group))
        for q, ix in sorted(self.idx.items()):
            buf = self._bufs.get(q)
            if buf is None or buf.shape[1] != rows.shape[1]:
                buf = torch.empty((ix.numel(), rows.shape[1]), dtype=rows.dtype, device=rows.device)
                self._bufs[q] = buf
            torch.index_select(rows, 0, ix, out=buf)
            self._work.append(dist.isend(buf, dst=q, group=self.group))

    def wait(self):
        for w in self._work:
            w.wait()
        self._work = []


class HostHaloExchange:
    """Ghost-row exchange staged through host memory over a CPU (gloo)
    process group, for ranks that share one GPU (tests): the send rows are
    gathered on the device and copied out, exchanged by gloo, and the
    received rows copied into the ghost block.  Every transfer is
    synchronous with the host, so no kernel ever waits on another rank's
    kernel (ranks on one GPU must not, B200_PROFILING.md)."""

    def __init__(self, part: LocalPart, device, group=None):
        import torch

        self.part = part
        self.group = group
        self.idx = {q: torch.as_tensor(ix, dtype=torch.int64, device=device) for q, ix in part.send_idx.items()}
        self._work = []
        self._recv = []

    def start(self, rows):
        import torch
        import torch.distributed as dist

        self._work, self._recv = [], []
        for q, (r0, cnt) in sorted(self.part.recv_range.items()):
            buf = torch.empty((cnt, rows.shape[1]), dtype=rows.dtype)
            self._recv.append((rows, r0, cnt, buf))
            self._work.append(dist.irecv(buf, src=q, group=self.group))
        for q, ix in sorted(self.idx.items()):
            buf = torch.index_select(rows, 0, ix).cpu()  # waits for the rows
            self._work.append(dist.isend(buf, dst=q, group=self.group))
            self._recv.append((None, 0, 0, buf))  # keep the send buffer alive

    def wait(self):
        for w in self._work:
            w.wait()
        for rows, r0, cnt, buf in self._recv:
            if rows is not None:
                rows[r0:r0 + cnt].copy_(buf)
        self._work, self._recv = [], []

    def allreduce(self, t, kind):
        """In place: kind 0 int64 MIN, 1 float64 SUM (through the host)."""
        import torch.distributed as dist

        host = t.cpu()
        dist.all_reduce(host, op=dist.ReduceOp.MIN if kind == 0 else dist.ReduceOp.SUM, group=self.group)
        t.copy_(host)


class NativeHaloExchange:
    """The same exchange through the library's NCCL halo (`hodg_halo_*`,
    csrc/halo.cu): one pack kernel plus grouped NCCL sends / receives on a
    communication stream, ghost rows received in place.  `start` orders the
    exchange after the work already queued on the current stream (the state
    rows are ready); `wait` makes the current stream wait for it, so the
    interior-face kernel runs while the halo is in flight.

    `nranks == 1` with the rank as its own peer is the single-GPU self test
    (tests/test_gpu_halo.py)."""

    def __init__(self, part: LocalPart, rs: int, rank: int, nranks: int, unique_id: bytes, device="cuda"):
        import ctypes as C

        import torch

        from . import _lib

        self.L = _lib.lib()
        self.part = part
        peers = sorted(set(part.send_idx) | set(part.recv_range))
        send_count = [len(part.send_idx.get(q, ())) for q in peers]
        rows = np.concatenate([np.asarray(part.send_idx[q], dtype=np.int32) for q in peers if q in part.send_idx]) \
            if part.send_idx else np.zeros(1, dtype=np.int32)
        recv_first = [part.recv_range.get(q, (0, 0))[0] for q in peers]
        recv_count = [part.recv_range.get(q, (0, 0))[1] for q in peers]
        arr = lambda v, t: np.ascontiguousarray(np.asarray(v, dtype=t))  # noqa: E731
        self._keep = (arr(peers, np.int32), arr(send_count, np.int64), arr(rows, np.int32),
                      arr(recv_first, np.int64), arr(recv_count, np.int64))
        uid = C.create_string_buffer(bytes(unique_id), 128)
        h = C.c_void_p()
        k = self._keep
        _lib.check(self.L.hodg_halo_create(int(nranks), int(rank), uid, len(peers), k[0].ctypes.data,
                                           k[1].ctypes.data, k[2].ctypes.data, k[3].ctypes.data, k[4].ctypes.data,
                                           int(rs), C.byref(h)), "hodg_halo_create")
        self.handle = h
        self.stream = torch.cuda.Stream(device=device)
        self._ready = torch.cuda.Event()
        self._done = torch.cuda.Event()

    @staticmethod
    def unique_id() -> bytes:
        import ctypes as C

        from . import _lib

        buf = C.create_string_buffer(128)
        _lib.check(_lib.lib().hodg_halo_unique_id(buf), "hodg_halo_unique_id")
        return buf.raw

    def start(self, rows):
        from . import _lib

        self._ready.record()
        self.stream.wait_event(self._ready)
        _lib.check(self.L.hodg_halo_exchange(self.handle, _lib.ptr(rows), _lib.stream_ptr(self.stream)),
                   "hodg_halo_exchange")
        self._done.record(self.stream)

    def wait(self):
        import torch

        torch.cuda.current_stream().wait_event(self._done)

    def allreduce(self, t, kind):
        """In place on the current stream: kind 0 int64 MIN, 1 float64 SUM."""
        from . import _lib

        _lib.check(self.L.hodg_halo_allreduce(self.handle, _lib.ptr(t), t.numel(), int(kind), _lib.stream_ptr()),
                   "hodg_halo_allreduce")

    def close(self):
        if getattr(self, "handle", None):
            self.L.hodg_halo_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
