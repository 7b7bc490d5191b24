// Multi-GPU plumbing behind the C ABI:
//  * hodg_partition_rcb: recursive coordinate bisection of element centroids
//    (host), bit-exact with paper_2209_01877_b200/partition.py:rcb_partition
//    and its restatement oracle/partition.py;
//  * hodg_halo_*: the per-stage ghost-row exchange over NCCL point-to-point
//    (NVLink / NVSwitch between the GPUs of a node): a pack kernel gathers the
//    owned rows each peer needs into one send block per peer, and the ghost
//    rows arrive straight in the state array (ghosts are ordered by
//    (owner, id), so each peer's rows are one contiguous block).
// NCCL is resolved at run time from the process's libnccl.so.2 (the one the
// host framework already loaded, e.g. PyTorch's), so the library has no
// link-time NCCL dependency.
#include <dlfcn.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <new>
#include <numeric>
#include <vector>

#include <nccl.h>

#include "../../include/hodg_b200.h"
#include "hodg_common.cuh"

extern int64_t hodg_count_launch(int64_t n);

namespace {

// ---------------------------------------------------------------------------
// RCB (partition.py:31-55): split along the first axis of maximal extent,
// order by (coordinate, id), first part gets (size * k1) // k points.
void rcb(const double* pts, std::vector<int64_t>& ids, int base, int k, int32_t* part) {
    if (k == 1) {
        for (int64_t i : ids) part[i] = base;
        return;
    }
    double lo[3], hi[3];
    for (int d = 0; d < 3; ++d) {
        lo[d] = pts[3 * ids[0] + d];
        hi[d] = lo[d];
    }
    for (int64_t i : ids)
        for (int d = 0; d < 3; ++d) {
            const double x = pts[3 * i + d];
            lo[d] = x < lo[d] ? x : lo[d];
            hi[d] = x > hi[d] ? x : hi[d];
        }
    int axis = 0;
    double best = hi[0] - lo[0];
    for (int d = 1; d < 3; ++d)
        if (hi[d] - lo[d] > best) {
            best = hi[d] - lo[d];
            axis = d;
        }
    std::sort(ids.begin(), ids.end(), [&](int64_t a, int64_t b) {
        const double xa = pts[3 * a + axis], xb = pts[3 * b + axis];
        return xa < xb || (xa == xb && a < b);
    });
    const int k1 = k / 2;
    const int64_t n1 = (int64_t(ids.size()) * k1) / k;
    std::vector<int64_t> left(ids.begin(), ids.begin() + n1), right(ids.begin() + n1, ids.end());
    ids.clear();
    ids.shrink_to_fit();
    rcb(pts, left, base, k1, part);
    rcb(pts, right, base + k1, k - k1, part);
}

// ---------------------------------------------------------------------------
// NCCL entry points, resolved once
struct Nccl {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    bool ok = false;
};

const Nccl& nccl() {
    static Nccl n;
    static bool tried = false;
    if (tried) return n;
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return n;
    n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(dlsym(h, "ncclGroupStart"));
    n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
    n.Send = reinterpret_cast<decltype(n.Send)>(dlsym(h, "ncclSend"));
    n.Recv = reinterpret_cast<decltype(n.Recv)>(dlsym(h, "ncclRecv"));
    n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(dlsym(h, "ncclAllReduce"));
    n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.GroupStart && n.GroupEnd && n.Send && n.Recv &&
           n.AllReduce;
    return n;
}

// pack: send block row k <- state row rows[k] (rs doubles per row, 16-byte
// vectors when rs is even)
__global__ void halo_pack_kernel(const double* __restrict__ state, const int32_t* __restrict__ rows, int64_t n,
                                 int rs, double* __restrict__ out) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;  // (row, pair) index
    const int half = rs / 2;
    if (rs % 2 == 0) {
        if (k >= n * half) return;
        const int64_t r = k / half, j = k - r * half;
        reinterpret_cast<double2*>(out)[r * half + j] =
            reinterpret_cast<const double2*>(state)[int64_t(rows[r]) * half + j];
    } else {
        if (k >= n * rs) return;
        const int64_t r = k / rs, j = k - r * rs;
        out[r * rs + j] = state[int64_t(rows[r]) * rs + j];
    }
}

}  // namespace

struct hodg_halo {
    ncclComm_t comm = nullptr;
    int nranks = 0, rank = 0, rs = 0;
    std::vector<int> peers;
    std::vector<int64_t> send_off, send_count, recv_first, recv_count;
    int32_t* rows = nullptr;  // device, concatenated send rows
    double* sendbuf = nullptr;
    int64_t n_send = 0;
};

extern "C" {

int hodg_partition_rcb(int64_t n, const double* points, int nparts, int32_t* part) {
    if (n < 1 || !points || !part || nparts < 1 || nparts > n) return HODG_EINVAL;
    std::vector<int64_t> ids(n);
    std::iota(ids.begin(), ids.end(), int64_t(0));
    rcb(points, ids, 0, nparts, part);
    return HODG_OK;
}

int hodg_halo_unique_id(void* id) {
    const Nccl& n = nccl();
    if (!id) return HODG_EINVAL;
    if (!n.ok) return HODG_ECUDA;
    ncclUniqueId u;
    if (n.GetUniqueId(&u) != ncclSuccess) return HODG_ECUDA;
    std::memcpy(id, &u, sizeof(u));
    return HODG_OK;
}

int hodg_halo_create(int nranks, int rank, const void* id, int npeers, const int32_t* peers,
                     const int64_t* send_count, const int32_t* send_rows, const int64_t* recv_first,
                     const int64_t* recv_count, int rs, hodg_halo** out) {
    if (!out || !id || nranks < 1 || rank < 0 || rank >= nranks || npeers < 0 || rs < 1) return HODG_EINVAL;
    if (npeers > 0 && (!peers || !send_count || !recv_first || !recv_count)) return HODG_EINVAL;
    const Nccl& n = nccl();
    if (!n.ok) return HODG_ECUDA;
    hodg_halo* h = new (std::nothrow) hodg_halo;
    if (!h) return HODG_EINVAL;
    h->nranks = nranks;
    h->rank = rank;
    h->rs = rs;
    int64_t off = 0;
    for (int p = 0; p < npeers; ++p) {
        if (peers[p] < 0 || peers[p] >= nranks || send_count[p] < 0 || recv_count[p] < 0 || recv_first[p] < 0) {
            delete h;
            return HODG_EINVAL;
        }
        h->peers.push_back(peers[p]);
        h->send_off.push_back(off);
        h->send_count.push_back(send_count[p]);
        h->recv_first.push_back(recv_first[p]);
        h->recv_count.push_back(recv_count[p]);
        off += send_count[p];
    }
    h->n_send = off;
    if (off > 0) {
        if (!send_rows || cudaMalloc(&h->rows, off * sizeof(int32_t)) != cudaSuccess ||
            cudaMalloc(&h->sendbuf, off * rs * sizeof(double)) != cudaSuccess ||
            cudaMemcpy(h->rows, send_rows, off * sizeof(int32_t), cudaMemcpyDefault) != cudaSuccess) {
            cudaFree(h->rows);
            cudaFree(h->sendbuf);
            delete h;
            return HODG_ECUDA;
        }
    }
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    if (n.CommInitRank(&h->comm, nranks, u, rank) != ncclSuccess) {
        cudaFree(h->rows);
        cudaFree(h->sendbuf);
        delete h;
        return HODG_ECUDA;
    }
    *out = h;
    return HODG_OK;
}

int hodg_halo_exchange(hodg_halo* h, double* state, void* stream) {
    if (!h || !state) return HODG_EINVAL;
    const Nccl& n = nccl();
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (h->n_send > 0) {
        hodg_count_launch(1);
        const int64_t items = h->rs % 2 == 0 ? h->n_send * (h->rs / 2) : h->n_send * h->rs;
        halo_pack_kernel<<<unsigned((items + 255) / 256), 256, 0, st>>>(state, h->rows, h->n_send, h->rs,
                                                                        h->sendbuf);
        if (cudaGetLastError() != cudaSuccess) return HODG_ECUDA;
    }
    if (n.GroupStart() != ncclSuccess) return HODG_ECUDA;
    // a failed Send / Recv still closes the group: an open group would batch
    // every later NCCL call on this thread (the dt / norm all-reduces) into a
    // group that never launches
    bool ok = true;
    for (size_t p = 0; p < h->peers.size() && ok; ++p) {
        if (h->recv_count[p] > 0)
            ok = n.Recv(state + h->recv_first[p] * h->rs, size_t(h->recv_count[p] * h->rs), ncclFloat64,
                        h->peers[p], h->comm, st) == ncclSuccess;
        if (ok && h->send_count[p] > 0)
            ok = n.Send(h->sendbuf + h->send_off[p] * h->rs, size_t(h->send_count[p] * h->rs), ncclFloat64,
                        h->peers[p], h->comm, st) == ncclSuccess;
    }
    const bool closed = n.GroupEnd() == ncclSuccess;
    return ok && closed ? HODG_OK : HODG_ECUDA;
}

int hodg_halo_allreduce(hodg_halo* h, void* buf, int64_t count, int kind, void* stream) {
    if (!h || !buf || count < 0 || kind < 0 || kind > 1) return HODG_EINVAL;
    const Nccl& n = nccl();
    // kind 0: int64 MIN (dt slots as double bit patterns: exact); 1: float64 SUM
    const ncclDataType_t t = kind == 0 ? ncclInt64 : ncclFloat64;
    const ncclRedOp_t op = kind == 0 ? ncclMin : ncclSum;
    return n.AllReduce(buf, buf, size_t(count), t, op, h->comm, static_cast<cudaStream_t>(stream)) == ncclSuccess
               ? HODG_OK
               : HODG_ECUDA;
}

int hodg_halo_destroy(hodg_halo* h) {
    if (!h) return HODG_OK;
    const Nccl& n = nccl();
    if (h->comm && n.ok) n.CommDestroy(h->comm);
    cudaFree(h->rows);
    cudaFree(h->sendbuf);
    delete h;
    return HODG_OK;
}

}  // extern "C"
