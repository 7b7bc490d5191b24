// Device mesh setup: the tetrahedral analogue of
// the reference's connectivity build (hodg/mesh.py:177-286, face discovery
// by sorted face keys) and the per-element / per-face geometry, on the GPU.
// Same numbering as the host builder paper_2209_01877_b200/mesh.py:
// build_tet_mesh: faces keyed by their ascending node triple, a face's id is
// the rank of its first traversal (element-major, slot order), the first
// traverser is the left element.  Integer outputs are bit-identical to the
// host build; the float geometry follows numpy's expression order and is
// compiled without FMA contraction, so it matches except where libm and
// CUDA differ (cbrt for h).
#include <cub/cub.cuh>

#include <cstdint>

#include "../../include/hodg_b200.h"

extern int64_t hodg_count_launch(int64_t n);

namespace {

constexpr int TPB = 256;
inline unsigned nb(int64_t n) { return unsigned((n + TPB - 1) / TPB); }
inline size_t al(size_t x) { return (x + 255) & ~size_t(255); }

__constant__ int FACE_LOCAL[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};

// slot s = 4 e + f: key of face f of element e (nodes ascending)
__global__ void face_key_kernel(int64_t ns, int64_t nn, const int32_t* __restrict__ tets,
                                unsigned long long* __restrict__ key, int32_t* __restrict__ slot) {
    const int64_t s = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= ns) return;
    const int64_t e = s >> 2;
    const int f = int(s & 3);
    const int64_t a = tets[4 * e + FACE_LOCAL[f][0]], b = tets[4 * e + FACE_LOCAL[f][1]],
                  c = tets[4 * e + FACE_LOCAL[f][2]];
    key[s] = (unsigned long long)((a * nn + b) * nn + c);
    slot[s] = int32_t(s);
}

// run heads of the sorted keys; more than two equal keys = non-manifold
__global__ void run_head_kernel(int64_t ns, const unsigned long long* __restrict__ ks, int32_t* __restrict__ head,
                                int* __restrict__ bad) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= ns) return;
    head[i] = (i == 0 || ks[i] != ks[i - 1]) ? 1 : 0;
    if (i >= 2 && ks[i] == ks[i - 2]) atomicExch(bad, 1);
}

// per run r (at its head i): first traversal slot and the second one
__global__ void run_info_kernel(int64_t ns, const int32_t* __restrict__ head, const int32_t* __restrict__ run,
                                const int32_t* __restrict__ order, const unsigned long long* __restrict__ ks,
                                int32_t* __restrict__ first, int32_t* __restrict__ second,
                                int32_t* __restrict__ rid) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= ns || !head[i]) return;
    const int32_t r = run[i] - 1;  // inclusive scan of heads - 1: run index
    first[r] = order[i];       // stable sort: the earliest traversal leads its run
    second[r] = (i + 1 < ns && ks[i + 1] == ks[i]) ? order[i + 1] : -1;
    rid[r] = r;
}

// face k (= rank of first traversal) from the runs sorted by first slot
__global__ void face_kernel(int64_t nf, const int32_t* __restrict__ fs_sorted, const int32_t* __restrict__ rid_sorted,
                            const int32_t* __restrict__ second, const int32_t* __restrict__ tets,
                            int32_t* __restrict__ face_rank, int32_t* __restrict__ face_cells,
                            int8_t* __restrict__ face_slots, int32_t* __restrict__ face_nodes) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= nf) return;
    const int32_t r = rid_sorted[k];
    face_rank[r] = int32_t(k);
    const int32_t ls = fs_sorted[k], rs = second[r];
    const int32_t le = ls >> 2, lf = ls & 3;
    face_cells[2 * k] = le;
    face_cells[2 * k + 1] = rs >= 0 ? (rs >> 2) : -1;
    face_slots[2 * k] = int8_t(lf);
    face_slots[2 * k + 1] = int8_t(rs >= 0 ? (rs & 3) : -1);
    for (int j = 0; j < 3; ++j) face_nodes[3 * k + j] = tets[4 * le + FACE_LOCAL[lf][j]];
}

// slot -> face id and side sign
__global__ void slot_face_kernel(int64_t ns, const int32_t* __restrict__ order, const int32_t* __restrict__ run,
                                 const int32_t* __restrict__ face_rank, const int32_t* __restrict__ face_cells,
                                 const int8_t* __restrict__ face_slots, int32_t* __restrict__ cell_faces,
                                 int8_t* __restrict__ cell_fsign) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= ns) return;
    const int32_t s = order[i];
    const int32_t f = face_rank[run[i] - 1];
    cell_faces[s] = f;
    cell_fsign[s] = (face_cells[2 * f] == (s >> 2) && face_slots[2 * f] == (s & 3)) ? 1 : -1;
}

// unit normal (left -> right), area (mesh.py build_tet_mesh, numpy order)
__global__ void face_geom_kernel(int64_t nf, const double* __restrict__ X, const int32_t* __restrict__ tets,
                                 const int32_t* __restrict__ face_nodes, const int32_t* __restrict__ face_cells,
                                 const int8_t* __restrict__ face_slots, double* __restrict__ normal,
                                 double* __restrict__ area, int* __restrict__ bad) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= nf) return;
    const double* A = X + 3 * int64_t(face_nodes[3 * k]);
    const double* B = X + 3 * int64_t(face_nodes[3 * k + 1]);
    const double* C = X + 3 * int64_t(face_nodes[3 * k + 2]);
    const double a0 = B[0] - A[0], a1 = B[1] - A[1], a2 = B[2] - A[2];
    const double b0 = C[0] - A[0], b1 = C[1] - A[1], b2 = C[2] - A[2];
    const double c0 = a1 * b2 - a2 * b1, c1 = a2 * b0 - a0 * b2, c2 = a0 * b1 - a1 * b0;
    // np.einsum("fd,fd->f") on this numpy sums (d0 + d2) + d1
    const double nrm = sqrt((c0 * c0 + c2 * c2) + c1 * c1);
    if (!(nrm > 0.0)) atomicExch(bad, 2);
    double n0 = c0 / nrm, n1 = c1 / nrm, n2 = c2 / nrm;
    const double* O = X + 3 * int64_t(tets[4 * face_cells[2 * k] + face_slots[2 * k]]);
    const double d = (n0 * (A[0] - O[0]) + n2 * (A[2] - O[2])) + n1 * (A[1] - O[1]);
    if (d < 0.0) {
        n0 = -n0;
        n1 = -n1;
        n2 = -n2;
    }
    normal[3 * k] = n0;
    normal[3 * k + 1] = n1;
    normal[3 * k + 2] = n2;
    area[k] = 0.5 * nrm;
}

// volume, centroid, h; neighbours
__global__ void elem_geom_kernel(int64_t n, const double* __restrict__ X, const int32_t* __restrict__ tets,
                                 const int32_t* __restrict__ cell_faces, const int32_t* __restrict__ face_cells,
                                 double* __restrict__ vol, double* __restrict__ centroid, double* __restrict__ h,
                                 int32_t* __restrict__ nbr, int* __restrict__ bad) {
    const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= n) return;
    const double* V[4];
    for (int j = 0; j < 4; ++j) V[j] = X + 3 * int64_t(tets[4 * e + j]);
    double a[3], b[3], c[3];
    for (int d = 0; d < 3; ++d) {
        a[d] = V[1][d] - V[0][d];
        b[d] = V[2][d] - V[0][d];
        c[d] = V[3][d] - V[0][d];
    }
    const double x0 = b[1] * c[2] - b[2] * c[1], x1 = b[2] * c[0] - b[0] * c[2], x2 = b[0] * c[1] - b[1] * c[0];
    const double v6 = (a[0] * x0 + a[2] * x2) + a[1] * x1;
    const double v = fabs(v6) / 6.0;
    if (!(v > 0.0)) atomicExch(bad, 3);
    vol[e] = v;
    for (int d = 0; d < 3; ++d) centroid[3 * e + d] = 0.25 * (V[0][d] + V[1][d] + V[2][d] + V[3][d]);
    h[e] = cbrt(v);
    for (int s = 0; s < 4; ++s) {
        const int32_t f = cell_faces[4 * e + s];
        const int32_t l = face_cells[2 * f], r = face_cells[2 * f + 1];
        nbr[4 * e + s] = l == int32_t(e) ? r : l;
    }
}

struct Work {
    unsigned long long *k0, *k1;
    int32_t *s0, *order, *head, *run, *first, *second, *rid, *fs_sorted, *rid_sorted, *face_rank;
    int* bad;
    void* cub;
    size_t cub_bytes;
};

size_t carve(int64_t n, char* base, Work* w) {
    const int64_t ns = 4 * n;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char* p = base ? base + off : nullptr;
        off += al(bytes);
        return p;
    };
    Work t;
    t.k0 = reinterpret_cast<unsigned long long*>(take(ns * 8));
    t.k1 = reinterpret_cast<unsigned long long*>(take(ns * 8));
    t.s0 = reinterpret_cast<int32_t*>(take(ns * 4));
    t.order = reinterpret_cast<int32_t*>(take(ns * 4));
    t.head = reinterpret_cast<int32_t*>(take(ns * 4));
    t.run = reinterpret_cast<int32_t*>(take(ns * 4));
    t.first = reinterpret_cast<int32_t*>(take(ns * 4));
    t.second = reinterpret_cast<int32_t*>(take(ns * 4));
    t.rid = reinterpret_cast<int32_t*>(take(ns * 4));
    t.fs_sorted = reinterpret_cast<int32_t*>(take(ns * 4));
    t.rid_sorted = reinterpret_cast<int32_t*>(take(ns * 4));
    t.face_rank = reinterpret_cast<int32_t*>(take(ns * 4));
    t.bad = reinterpret_cast<int*>(take(16));
    size_t a = 0, b = 0, c = 0;
    const int nsi = int(ns > 0 ? ns : 1);
    cub::DeviceRadixSort::SortPairs(nullptr, a, t.k0, t.k1, t.s0, t.order, nsi);
    cub::DeviceRadixSort::SortPairs(nullptr, b, t.first, t.fs_sorted, t.rid, t.rid_sorted, nsi);
    cub::DeviceScan::InclusiveSum(nullptr, c, t.head, t.run, nsi);
    t.cub_bytes = a > b ? (a > c ? a : c) : (b > c ? b : c);
    t.cub = take(t.cub_bytes);
    if (w) *w = t;
    return off + 256;
}


// Element geometry records and modal-transform maps on the GPU: the device
// twin of paper_2209_01877_b200/geometry.py:compute_geometry (egeo, econv),
// which replaces the reference's per-cell tables (hodg/geometry.py:120-220).
// J[d][k] = (V_{k+1} - V_0)[d]; J^-1 by the adjugate over the determinant
// (the host build uses LAPACK's LU: the two agree to a few ulp).  fc, J/h and
// J^-1 h are single roundings in numpy's order, bit-identical to the host's
// given the same J^-1.  egeo is tile-major [tile][16][T]; the caller zeroes it.
__global__ void elem_record_kernel(int64_t n, int T, const double* __restrict__ X, const int32_t* __restrict__ tets,
                                   const double* __restrict__ vol, const double* __restrict__ hh,
                                   const double* __restrict__ farea, const int32_t* __restrict__ cell_faces,
                                   const int8_t* __restrict__ fsign, double* __restrict__ egeo,
                                   double* __restrict__ econv, int* __restrict__ bad) {
    const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= n) return;
    double V[4][3];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int d = 0; d < 3; ++d) V[k][d] = X[int64_t(tets[e * 4 + k]) * 3 + d];
    double J[3][3];
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int k = 0; k < 3; ++k) J[d][k] = V[k + 1][d] - V[0][d];
    double C[3][3];  // cofactors
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
            C[i][j] = J[i1][j1] * J[i2][j2] - J[i1][j2] * J[i2][j1];
        }
    const double det = J[0][0] * C[0][0] + J[0][1] * C[0][1] + J[0][2] * C[0][2];
    if (!(fabs(det) > 0.0)) {
        atomicMax(bad, 3);
        return;
    }
    const double h = hh[e], v = vol[e];
    const int64_t base = (e / T) * 16 * T + (e % T);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const double ji = C[j][i] / det;
            egeo[base + (i * 3 + j) * int64_t(T)] = ji;
            econv[e * 18 + i * 3 + j] = J[i][j] / h;
            econv[e * 18 + 9 + i * 3 + j] = ji * h;
        }
#pragma unroll
    for (int s = 0; s < 4; ++s)
        egeo[base + (9 + s) * int64_t(T)] = double(fsign[e * 4 + s]) * farea[cell_faces[e * 4 + s]] / v;
    egeo[base + 13 * int64_t(T)] = h;
    egeo[base + 14 * int64_t(T)] = v;
}

}  // namespace

extern "C" {

int64_t hodg_mesh_setup_work_bytes(int64_t n_elems) {
    if (n_elems <= 0 || 4 * n_elems >= (int64_t(1) << 31)) return -1;
    return int64_t(carve(n_elems, nullptr, nullptr));
}

int hodg_mesh_setup(int64_t n_nodes, int64_t n_elems, const double* X, const int32_t* tets, int32_t* face_cells,
                    int8_t* face_slots, int32_t* face_nodes, double* face_normal, double* face_area,
                    int32_t* cell_faces, int8_t* cell_fsign, int32_t* cell_neighbors, double* cell_volume,
                    double* cell_centroid, double* cell_h, int64_t* n_faces_out, void* work, void* stream) {
    if (n_nodes <= 0 || n_elems <= 0 || !X || !tets || !face_cells || !face_slots || !face_nodes || !face_normal ||
        !face_area || !cell_faces || !cell_fsign || !cell_neighbors || !cell_volume || !cell_centroid || !cell_h ||
        !n_faces_out || !work)
        return HODG_EINVAL;
    // the packed key (a nn + b) nn + c must fit in 64 bits
    if (n_nodes >= (int64_t(1) << 21) || 4 * n_elems >= (int64_t(1) << 31)) return HODG_EINVAL;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(work) + 255) & ~uintptr_t(255));
    Work w;
    carve(n_elems, base, &w);
    const int64_t ns = 4 * n_elems;
    int end_bit = 1;
    const unsigned long long kmax = (unsigned long long)n_nodes * n_nodes * n_nodes;
    while (end_bit < 64 && ((unsigned long long)1 << end_bit) <= kmax) ++end_bit;
    cudaMemsetAsync(w.bad, 0, sizeof(int), st);
    face_key_kernel<<<nb(ns), TPB, 0, st>>>(ns, n_nodes, tets, w.k0, w.s0);
    size_t tb = w.cub_bytes;
    if (cub::DeviceRadixSort::SortPairs(w.cub, tb, w.k0, w.k1, w.s0, w.order, int(ns), 0, end_bit, st) !=
        cudaSuccess)
        return HODG_ECUDA;
    run_head_kernel<<<nb(ns), TPB, 0, st>>>(ns, w.k1, w.head, w.bad);
    tb = w.cub_bytes;
    if (cub::DeviceScan::InclusiveSum(w.cub, tb, w.head, w.run, int(ns), st) != cudaSuccess) return HODG_ECUDA;
    int32_t last_run = 0;
    cudaMemcpyAsync(&last_run, w.run + ns - 1, 4, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return HODG_ECUDA;
    const int64_t nf = last_run;
    run_info_kernel<<<nb(ns), TPB, 0, st>>>(ns, w.head, w.run, w.order, w.k1, w.first, w.second, w.rid);
    int bits = 1;
    while (bits < 32 && (int64_t(1) << bits) <= ns) ++bits;
    tb = w.cub_bytes;
    if (cub::DeviceRadixSort::SortPairs(w.cub, tb, w.first, w.fs_sorted, w.rid, w.rid_sorted, int(nf), 0, bits,
                                        st) != cudaSuccess)
        return HODG_ECUDA;
    face_kernel<<<nb(nf), TPB, 0, st>>>(nf, w.fs_sorted, w.rid_sorted, w.second, tets, w.face_rank, face_cells,
                                        face_slots, face_nodes);
    slot_face_kernel<<<nb(ns), TPB, 0, st>>>(ns, w.order, w.run, w.face_rank, face_cells, face_slots, cell_faces,
                                             cell_fsign);
    face_geom_kernel<<<nb(nf), TPB, 0, st>>>(nf, X, tets, face_nodes, face_cells, face_slots, face_normal, face_area,
                                             w.bad);
    elem_geom_kernel<<<nb(n_elems), TPB, 0, st>>>(n_elems, X, tets, cell_faces, face_cells, cell_volume,
                                                  cell_centroid, cell_h, cell_neighbors, w.bad);
    int bad = 0;
    cudaMemcpyAsync(&bad, w.bad, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return HODG_ECUDA;
    hodg_count_launch(9);
    *n_faces_out = bad ? -int64_t(bad) : nf;
    return bad ? HODG_ETOPOLOGY : HODG_OK;
}

int hodg_element_records(int64_t n_elems, int order, const double* X, const int32_t* tets, const double* cell_volume,
                         const double* cell_h, const double* face_area, const int32_t* cell_faces,
                         const int8_t* cell_fsign, double* egeo, double* econv, int32_t* flag, void* stream) {
    if (n_elems <= 0 || !X || !tets || !cell_volume || !cell_h || !face_area || !cell_faces || !cell_fsign || !egeo ||
        !econv || !flag)
        return HODG_EINVAL;
    const int T = hodg_elem_tile(order);
    if (T <= 0) return HODG_EINVAL;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t nt = (n_elems + T - 1) / T;
    if (cudaMemsetAsync(egeo, 0, size_t(nt) * 16 * T * sizeof(double), st) != cudaSuccess ||
        cudaMemsetAsync(flag, 0, sizeof(int32_t), st) != cudaSuccess)
        return HODG_ECUDA;
    elem_record_kernel<<<nb(n_elems), TPB, 0, st>>>(n_elems, T, X, tets, cell_volume, cell_h, face_area, cell_faces,
                                                    cell_fsign, egeo, econv, reinterpret_cast<int*>(flag));
    hodg_count_launch(1);
    int bad = 0;
    cudaMemcpyAsync(&bad, flag, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return HODG_ECUDA;
    return bad ? HODG_ETOPOLOGY : HODG_OK;
}

}  // extern "C"
