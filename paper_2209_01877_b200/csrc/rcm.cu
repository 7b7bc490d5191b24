// Device Reverse Cuthill-McKee, bit-exact with the reference
// (hodg/renumber.py:135-208).
//
// The reference runs a sequential queue BFS that appends each vertex's
// unvisited neighbours in (degree, id) order.  Its level-synchronous
// equivalent: level L+1 is the set of unvisited neighbours of level L; a
// vertex's parent is the earliest-positioned level-L vertex adjacent to it
// (atomicMin on positions); level L+1 is ordered by the key
// (parent position, degree, id) -- which is exactly the sequential queue
// order.  The George-Liu pseudo-peripheral start (renumber.py:153-168) and
// the component seeding in ascending smallest id (renumber.py:184-188) are
// reproduced with order-independent level BFS + (degree, id) argmin
// reductions.  Sorting each level uses a 64-bit packed key and CUB's radix
// sort (header library from the CUDA toolkit).
#include <cub/device/device_radix_sort.cuh>

#include <cstdint>
#include <vector>

#include "../../include/hodg_b200.h"

namespace {

constexpr int TPB = 256;

struct Work {
    int32_t* level;
    int32_t* deg;
    int32_t* members;
    int32_t* front;
    int32_t* next;
    int64_t* pos;
    int64_t* parent;
    unsigned long long* keys;
    unsigned long long* keys2;
    unsigned long long* scal;  // [0] counter, [1] argmin key, [2] min unvisited
    void* cub;
    size_t cub_bytes;
};

inline size_t al(size_t x) { return (x + 255) & ~size_t(255); }

size_t cub_bytes_for(int64_t n) {
    size_t b = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, b, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                   int(n > 0 ? n : 1), 0, 64);
    return b;
}

bool carve(void* base, int64_t n, Work& w) {
    char* p = static_cast<char*>(base);
    const size_t n4 = al(size_t(n) * 4), n8 = al(size_t(n) * 8);
    w.level = reinterpret_cast<int32_t*>(p); p += n4;
    w.deg = reinterpret_cast<int32_t*>(p); p += n4;
    w.members = reinterpret_cast<int32_t*>(p); p += n4;
    w.front = reinterpret_cast<int32_t*>(p); p += n4;
    w.next = reinterpret_cast<int32_t*>(p); p += n4;
    w.pos = reinterpret_cast<int64_t*>(p); p += n8;
    w.parent = reinterpret_cast<int64_t*>(p); p += n8;
    w.keys = reinterpret_cast<unsigned long long*>(p); p += n8;
    w.keys2 = reinterpret_cast<unsigned long long*>(p); p += n8;
    w.scal = reinterpret_cast<unsigned long long*>(p); p += al(64);
    w.cub = p;
    w.cub_bytes = cub_bytes_for(n);
    return true;
}

__global__ void init_kernel(int64_t n, const int64_t* __restrict__ indptr, Work w) {
    const int64_t v = int64_t(blockIdx.x) * TPB + threadIdx.x;
    if (v >= n) return;
    w.deg[v] = int32_t(indptr[v + 1] - indptr[v]);
    w.level[v] = -1;
    w.pos[v] = -1;
    w.parent[v] = INT64_MAX;
}

__global__ void min_unvisited_kernel(int64_t n, int64_t from, Work w) {
    const int64_t v = from + int64_t(blockIdx.x) * TPB + threadIdx.x;
    if (v < n && w.pos[v] < 0) atomicMin(&w.scal[2], (unsigned long long)v);
}

// expand one level: frontier -> next (unordered), levels only
__global__ void expand_kernel(const int64_t* __restrict__ indptr, const int64_t* __restrict__ indices, int32_t nf,
                              int32_t lvl, Work w, int32_t* __restrict__ front, int32_t* __restrict__ next) {
    const int i = blockIdx.x * TPB + threadIdx.x;
    if (i >= nf) return;
    const int32_t u = front[i];
    for (int64_t k = indptr[u]; k < indptr[u + 1]; ++k) {
        const int32_t x = int32_t(indices[k]);
        if (atomicCAS(&w.level[x], -1, lvl + 1) == -1) {
            const unsigned long long slot = atomicAdd(&w.scal[0], 1ull);
            next[slot] = x;
        }
    }
}

// ordered expansion: parent position = min position of a level-L neighbour
__global__ void expand_ordered_kernel(const int64_t* __restrict__ indptr, const int64_t* __restrict__ indices,
                                      int32_t nf, int32_t lvl, Work w, const int32_t* __restrict__ front,
                                      int32_t* __restrict__ next) {
    const int i = blockIdx.x * TPB + threadIdx.x;
    if (i >= nf) return;
    const int32_t u = front[i];
    const int64_t pu = w.pos[u];
    for (int64_t k = indptr[u]; k < indptr[u + 1]; ++k) {
        const int32_t x = int32_t(indices[k]);
        const int32_t lx = w.level[x];
        if (lx == -1 || lx == lvl + 1) {
            atomicMin(reinterpret_cast<unsigned long long*>(&w.parent[x]), (unsigned long long)pu);
            if (lx == -1 && atomicCAS(&w.level[x], -1, lvl + 1) == -1) {
                const unsigned long long slot = atomicAdd(&w.scal[0], 1ull);
                next[slot] = x;
            }
        }
    }
}

__global__ void make_keys_kernel(int32_t nn, const int32_t* __restrict__ next, Work w, int64_t base, int bn, int bd) {
    const int i = blockIdx.x * TPB + threadIdx.x;
    if (i >= nn) return;
    const int32_t x = next[i];
    const unsigned long long rel = (unsigned long long)(w.parent[x] - base);
    w.keys[i] = (rel << (bd + bn)) | ((unsigned long long)w.deg[x] << bn) | (unsigned long long)x;
}

__global__ void place_kernel(int32_t nn, const unsigned long long* __restrict__ sorted, int bn, Work w, int64_t off,
                             int64_t* __restrict__ order, int32_t* __restrict__ front) {
    const int i = blockIdx.x * TPB + threadIdx.x;
    if (i >= nn) return;
    const int32_t x = int32_t(sorted[i] & ((1ull << bn) - 1));
    order[off + i] = x;
    w.pos[x] = off + i;
    front[i] = x;
}

__global__ void argmin_deg_id_kernel(int32_t nn, const int32_t* __restrict__ list, Work w, int bn) {
    const int i = blockIdx.x * TPB + threadIdx.x;
    if (i >= nn) return;
    const int32_t x = list[i];
    atomicMin(&w.scal[1], ((unsigned long long)w.deg[x] << bn) | (unsigned long long)x);
}

__global__ void reset_levels_kernel(int32_t nn, const int32_t* __restrict__ list, Work w) {
    const int i = blockIdx.x * TPB + threadIdx.x;
    if (i < nn) w.level[list[i]] = -1;
}

__global__ void copy_list_kernel(int32_t nn, const int32_t* __restrict__ src, int32_t* __restrict__ dst, int32_t off) {
    const int i = blockIdx.x * TPB + threadIdx.x;
    if (i < nn) dst[off + i] = src[i];
}

__global__ void set_scalar_kernel(unsigned long long* p, unsigned long long v) { *p = v; }

__global__ void seed_kernel(int32_t r, int64_t off, Work w, int64_t* order, int32_t* front) {
    w.level[r] = 0;
    w.pos[r] = off;
    order[off] = r;
    front[0] = r;
}

__global__ void finish_kernel(int64_t n, const int64_t* __restrict__ order, int64_t* __restrict__ forward,
                              int64_t* __restrict__ inverse) {
    const int64_t i = int64_t(blockIdx.x) * TPB + threadIdx.x;
    if (i >= n) return;
    const int64_t v = order[n - 1 - i];  // reverse
    inverse[i] = v;
    forward[v] = i;
}

inline unsigned nb(int64_t k) { return unsigned((k + TPB - 1) / TPB); }

int bits_for(int64_t x) {
    int b = 1;
    while ((1ll << b) <= x) ++b;
    return b;
}

struct Ctx {
    const int64_t* indptr;
    const int64_t* indices;
    Work w;
    cudaStream_t st;
    int64_t launches = 0;
    bool fail = false;

    unsigned long long read(int k) {
        unsigned long long v = 0;
        if (cudaMemcpyAsync(&v, &w.scal[k], 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            fail = true;
        return v;
    }
    void setc(int k, unsigned long long v) {
        set_scalar_kernel<<<1, 1, 0, st>>>(&w.scal[k], v);
        ++launches;
    }

    // level BFS from r over one component (levels must be -1 there); returns
    // eccentricity; optional: the member list (collect) and the last level in w.front
    int32_t bfs(int32_t r, bool collect, int32_t* n_members, int32_t* n_last) {
        int32_t nf = 1, lvl = 0, total = 0;
        seed_levels(r);
        int32_t* front = w.front;
        int32_t* next = w.next;
        if (collect) {
            copy_list_kernel<<<1, TPB, 0, st>>>(1, front, w.members, 0);
            ++launches;
        }
        total = 1;
        for (;;) {
            setc(0, 0);
            expand_kernel<<<nb(nf), TPB, 0, st>>>(indptr, indices, nf, lvl, w, front, next);
            ++launches;
            const int32_t nn = int32_t(read(0));
            if (fail) return -1;
            if (nn == 0) break;
            if (collect) {
                copy_list_kernel<<<nb(nn), TPB, 0, st>>>(nn, next, w.members, total);
                ++launches;
            }
            total += nn;
            std::swap(front, next);
            nf = nn;
            ++lvl;
        }
        if (front != w.front) {  // keep the last level in w.front
            copy_list_kernel<<<nb(nf), TPB, 0, st>>>(nf, front, w.front, 0);
            ++launches;
        }
        if (n_members) *n_members = total;
        if (n_last) *n_last = nf;
        return lvl;
    }

    void seed_levels(int32_t r) {
        // level[r] = 0, front = [r]; pos untouched
        int32_t* front = w.front;
        level_seed_kernel_launch(r, front);
    }
    void level_seed_kernel_launch(int32_t r, int32_t* front);
};

__global__ void level_seed_kernel(int32_t r, Work w, int32_t* front) {
    w.level[r] = 0;
    front[0] = r;
}

void Ctx::level_seed_kernel_launch(int32_t r, int32_t* front) {
    level_seed_kernel<<<1, 1, 0, st>>>(r, w, front);
    ++launches;
}

}  // namespace

int64_t hodg_rcm_work_bytes_impl(int64_t n, int64_t nnz) {
    (void)nnz;
    if (n <= 0) return 256;
    return int64_t(5 * al(size_t(n) * 4) + 4 * al(size_t(n) * 8) + al(64) + al(cub_bytes_for(n)) + 256);
}

int hodg_rcm_impl(int64_t n, const int64_t* indptr, const int64_t* indices, int64_t* forward, int64_t* inverse,
                  void* work, cudaStream_t st, int64_t* launches) {
    if (n < 0 || (n > 0 && (!indptr || !forward || !inverse || !work))) return HODG_EINVAL;
    if (n == 0) return HODG_OK;
    if (n >= (1ll << 31)) return HODG_EINVAL;
    Ctx cx;
    cx.indptr = indptr;
    cx.indices = indices;
    cx.st = st;
    carve(work, n, cx.w);
    Work& w = cx.w;
    init_kernel<<<nb(n), TPB, 0, st>>>(n, indptr, w);
    ++cx.launches;
    // key widths
    int64_t maxdeg = 0;
    {
        std::vector<int64_t> ip(size_t(n) + 1);
        if (cudaMemcpyAsync(ip.data(), indptr, (size_t(n) + 1) * 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return HODG_ECUDA;
        for (int64_t v = 0; v < n; ++v) maxdeg = std::max(maxdeg, ip[size_t(v) + 1] - ip[size_t(v)]);
    }
    const int bn = bits_for(n);
    const int bd = bits_for(maxdeg);
    if (2 * bn + bd > 64) return HODG_EINVAL;
    // `order` reuses the inverse array until the final reversal
    int64_t* order = inverse;
    int64_t out = 0;
    int64_t from = 0;
    while (out < n) {
        cx.setc(2, ~0ull);
        min_unvisited_kernel<<<nb(n - from), TPB, 0, st>>>(n, from, w);
        ++cx.launches;
        const int32_t seed = int32_t(cx.read(2));
        if (cx.fail) return HODG_ECUDA;
        from = seed;
        // component of the seed
        int32_t nc = 0;
        cx.bfs(seed, true, &nc, nullptr);
        if (cx.fail) return HODG_ECUDA;
        // start: argmin (degree, id) over the component
        cx.setc(1, ~0ull);
        argmin_deg_id_kernel<<<nb(nc), TPB, 0, st>>>(nc, w.members, w, bn);
        ++cx.launches;
        int32_t r = int32_t(cx.read(1) & ((1ull << bn) - 1));
        // George-Liu double BFS
        for (;;) {
            reset_levels_kernel<<<nb(nc), TPB, 0, st>>>(nc, w.members, w);
            ++cx.launches;
            int32_t nlast = 0;
            const int32_t ecc = cx.bfs(r, false, nullptr, &nlast);
            cx.setc(1, ~0ull);
            argmin_deg_id_kernel<<<nb(nlast), TPB, 0, st>>>(nlast, w.front, w, bn);
            ++cx.launches;
            const int32_t cand = int32_t(cx.read(1) & ((1ull << bn) - 1));
            reset_levels_kernel<<<nb(nc), TPB, 0, st>>>(nc, w.members, w);
            ++cx.launches;
            const int32_t ecc2 = cx.bfs(cand, false, nullptr, nullptr);
            if (cx.fail) return HODG_ECUDA;
            reset_levels_kernel<<<nb(nc), TPB, 0, st>>>(nc, w.members, w);
            ++cx.launches;
            if (ecc2 > ecc) r = cand;
            else break;
        }
        // ordered BFS (Cuthill-McKee) from r
        seed_kernel<<<1, 1, 0, st>>>(r, out, w, order, w.front);
        ++cx.launches;
        int64_t fstart = out;
        int32_t nf = 1, lvl = 0;
        int64_t placed = 1;
        for (;;) {
            cx.setc(0, 0);
            expand_ordered_kernel<<<nb(nf), TPB, 0, st>>>(indptr, indices, nf, lvl, w, w.front, w.next);
            ++cx.launches;
            const int32_t nn = int32_t(cx.read(0));
            if (cx.fail) return HODG_ECUDA;
            if (nn == 0) break;
            make_keys_kernel<<<nb(nn), TPB, 0, st>>>(nn, w.next, w, fstart, bn, bd);
            ++cx.launches;
            size_t tb = w.cub_bytes;
            if (cub::DeviceRadixSort::SortKeys(w.cub, tb, w.keys, w.keys2, nn, 0, 2 * bn + bd, st) != cudaSuccess)
                return HODG_ECUDA;
            ++cx.launches;
            place_kernel<<<nb(nn), TPB, 0, st>>>(nn, w.keys2, bn, w, fstart + nf, order, w.front);
            ++cx.launches;
            fstart += nf;
            placed += nn;
            nf = nn;
            ++lvl;
        }
        out += placed;
    }
    // order currently aliases `inverse`; reverse through `forward` as scratch
    if (cudaMemcpyAsync(forward, order, size_t(n) * 8, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return HODG_ECUDA;
    finish_kernel<<<nb(n), TPB, 0, st>>>(n, forward, reinterpret_cast<int64_t*>(w.keys), inverse);
    ++cx.launches;
    // finish wrote forward-map into keys scratch; copy to forward
    if (cudaMemcpyAsync(forward, w.keys, size_t(n) * 8, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return HODG_ECUDA;
    if (launches) *launches = cx.launches;
    return cudaGetLastError() == cudaSuccess ? HODG_OK : HODG_ECUDA;
}

// ---------------------------------------------------------------------------
// Face re-sort of apply_permutation (hodg/renumber.py:224-231): stable sort
// of the faces by the packed key (min, max) of the new incident element ids
// (boundary faces use right = left).  A stable LSD radix sort of the key with
// the old face id as the value reproduces numpy's lexsort((ids, kmax, kmin)).
namespace {
__global__ void face_keys_kernel(int64_t nf, int64_t n, const int64_t* __restrict__ lr,
                                 unsigned long long* __restrict__ keys, int64_t* __restrict__ ids) {
    const int64_t f = int64_t(blockIdx.x) * TPB + threadIdx.x;
    if (f >= nf) return;
    const int64_t l = lr[2 * f];
    const int64_t r = lr[2 * f + 1] >= 0 ? lr[2 * f + 1] : l;
    const int64_t lo = l < r ? l : r, hi = l < r ? r : l;
    keys[f] = (unsigned long long)lo * (unsigned long long)(n + 1) + (unsigned long long)hi;
    ids[f] = f;
}
}  // namespace

int64_t hodg_face_sort_work_bytes(int64_t nf) {
    size_t b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                    (int64_t*)nullptr, (int64_t*)nullptr, int(nf > 0 ? nf : 1), 0, 64);
    return int64_t(3 * al(size_t(nf) * 8) + al(b) + 256);
}

extern int64_t hodg_count_launch(int64_t n);

extern "C" int hodg_face_sort(int64_t nf, int64_t n, const int64_t* lr, int64_t* order, void* work,
                              void* stream) {
    if (nf <= 0 || n <= 0 || !lr || !order || !work) return HODG_EINVAL;
    if (nf >= (1ll << 31)) return HODG_EINVAL;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    char* p = static_cast<char*>(work);
    auto* k0 = reinterpret_cast<unsigned long long*>(p);
    p += al(size_t(nf) * 8);
    auto* k1 = reinterpret_cast<unsigned long long*>(p);
    p += al(size_t(nf) * 8);
    auto* ids = reinterpret_cast<int64_t*>(p);
    p += al(size_t(nf) * 8);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, ids, order, int(nf), 0, 64, st);
    face_keys_kernel<<<nb(nf), TPB, 0, st>>>(nf, n, lr, k0, ids);
    int end_bit = 1;  // significant key bits: key < (n + 1)^2
    while (end_bit < 64 && ((unsigned long long)1 << end_bit) <= (unsigned long long)(n + 1) * (unsigned long long)(n + 1))
        ++end_bit;
    if (cub::DeviceRadixSort::SortPairs(p, tb, k0, k1, ids, order, int(nf), 0, end_bit, st) != cudaSuccess)
        return HODG_ECUDA;
    hodg_count_launch(2);
    return cudaGetLastError() == cudaSuccess ? HODG_OK : HODG_ECUDA;
}
