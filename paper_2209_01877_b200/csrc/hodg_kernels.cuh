// Per-order tetrahedral DG kernels.  Included once per polynomial order by
// hodg_p{0..3}.cu after the order's constant tables, with
//   ORDER, NB, NQV, NQF and the table macros VB_D/VB_F, VD_D/VD_F,
//   FB_D/FB_F, FG_D/FG_F, MINV_T, MEAN_T
// defined.  See DESIGN.md for the formulation: every element works in the
// reference-element monomial basis m_i(eta), so the reference's per-cell
// tables (hodg/geometry.py:33-51) collapse into compile-time constants and
// the per-element data is 16 doubles (J^-1, sgn*area/vol per face, h, vol).

#include <cstdlib>
#include <utility>

#include "hodg_common.cuh"

#define HODG_CAT_(a, b) a##b
#define HODG_CAT(a, b) HODG_CAT_(a, b)
// FP32 tables as compile-time constants (each value an FFMA immediate) or
// as __constant__ arrays (a uniform-register load per 4 values)
#ifndef HODG_F32_IMM
#define HODG_F32_IMM 1
#endif
#if HODG_F32_IMM
#define HODG_TABF(NAME) HODG_CAT(NAME, _FX)
#else
#define HODG_TABF(NAME) HODG_CAT(NAME, _F)
#endif
#define TAB(NAME, T, k) (sizeof(T) == 8 ? (T)HODG_CAT(NAME, _D)[(k)] : (T)HODG_TABF(NAME)[(k)])

namespace hodg {
namespace HODG_CAT(ord, ORDER) {

constexpr int RS = (5 * NB + 1) & ~1;        // state row stride (doubles)
constexpr int RSF = (5 * NB + 3) & ~3;       // FP32 shadow row stride (floats; 16-byte rows)
// row stride of a state array of element type R
template <typename R>
__host__ __device__ constexpr int rstride() {
    return sizeof(R) == 8 ? RS : RSF;
}
#ifndef HODG_NG3
#define HODG_NG3 4
#endif
#ifndef HODG_NG2
#define HODG_NG2 2
#endif
#ifndef HODG_NG1
#define HODG_NG1 2
#endif
// face qp groups per side thread (phase 1): bounds the trace accumulators
constexpr int NG = ORDER == 3 ? HODG_NG3 : (ORDER == 2 ? HODG_NG2 : (ORDER == 1 ? HODG_NG1 : 1));
constexpr int QPT = (NQF + NG - 1) / NG;     // face qps per phase-1 thread
#ifndef HODG_FACE_THREADS
#define HODG_FACE_THREADS 128
#endif
constexpr int FACE_THREADS = HODG_FACE_THREADS;
#ifndef HODG_ROE_PAIRS
#define HODG_ROE_PAIRS 1
#endif
#ifndef HODG_FACE_MINB_F
// mixed-precision face kernel: CTAs per SM of the register budget (6: 80
// registers; P2 with the FFMA2 trace pairs: 5 at 96 registers, no spills --
// face 0.326 -> 0.294 ms, where 6 spills 40 bytes)
#define HODG_FACE_MINB_F (ORDER == 2 ? 5 : 6)
#endif
#ifndef HODG_FACE_MINB
#define HODG_FACE_MINB (ORDER == 2 ? 4 : 5)
#endif
// CTA element kernel, face-ordered records: 16-byte cp.async chunks (1) or
// TMA copies (0: gather4 / one per record).  FP64: TMA gather4 is faster;
// FP32: cp.async (P2 element kernel 0.346 -> 0.335 ms, P1 0.201 -> 0.192 ms
// at C1M) -- its records' padded stride keeps the reads conflict-free,
// which gather4's 128-byte groups would not
#ifndef HODG_ELEM_CPASYNC
#define HODG_ELEM_CPASYNC 0
#endif
#ifndef HODG_ELEM_CPASYNC_F
#define HODG_ELEM_CPASYNC_F 1
#endif
#ifndef HODG_FACE_CPASYNC
#define HODG_FACE_CPASYNC 0  // state rows by per-thread cp.async chunks (0: one TMA bulk copy per row; faster)
#endif
constexpr int RP = HODG_ROE_PAIRS;  // Riemann problems per thread per phase-2 iteration (1 measured fastest)
constexpr int FT = FACE_THREADS / (2 * NG);  // faces per CTA (32 for P1-P3)
constexpr int FBS = NQF * NB + 1;            // padded per-slot stride of the smem trace table
// element kernel: E elements per CTA, thread (v, h, e) -- variable v, basis
// part h of H (each thread owns NB/H basis functions of its (v, e); H > 1
// halves the per-thread registers at P3 so twice the warps fit per SM)
#ifndef HODG_H2
#define HODG_H2 1
#endif
#ifndef HODG_H3
#define HODG_H3 2
#endif
constexpr int H = (ORDER == 3) ? HODG_H3 : (ORDER == 2 ? HODG_H2 : 1);
#ifndef HODG_E2
#define HODG_E2 32
#endif
#ifndef HODG_E1
#define HODG_E1 32
#endif
// P1 and P2 run the warp-group element kernel (hodg_elem_warp.cuh): G = 6
// elements per warp, lane (e, v); its element tile is the warp's group
#ifndef HODG_WARP_ELEM_P1
#define HODG_WARP_ELEM_P1 0
#endif
#ifndef HODG_WARP_ELEM_P2
#define HODG_WARP_ELEM_P2 0
#endif
constexpr bool WARP_ELEM = (ORDER == 1 && HODG_WARP_ELEM_P1) || (ORDER == 2 && HODG_WARP_ELEM_P2);
// volume integral of the CTA element kernel through the moments of the
// physical flux (hodg_elem_warp.cuh explains the identity); H == 1 only
#ifndef HODG_MOMENTS
#define HODG_MOMENTS 1
#endif
constexpr int NBL = ORDER * (ORDER + 1) * (ORDER + 2) / 6;  // monomials of degree < ORDER
constexpr bool MOMENTS = HODG_MOMENTS && H == 1 && ORDER >= 1;
constexpr int G = 6;
constexpr int E = WARP_ELEM ? G
                            : ((ORDER >= 3) ? (H > 1 ? 32 : 16) : (ORDER == 2 ? HODG_E2 : (ORDER == 1 ? HODG_E1 : 64)));
constexpr int NH = NB / H;
static_assert(NB % H == 0 && (H == 1 || E >= 32) && 5 * H <= 15, "basis split layout");
constexpr int ETHREADS = 5 * E * H;
#ifndef HODG_PDL
// face and element kernels launched as programmatic dependents (griddepcontrol)
// on meshes of at most HODG_PDL_MAX_ELEMS elements: measured +2% per step on a
// 125k-element partition, -1.5% at 1M elements (the kernels always carry the
// griddepcontrol instructions; they are no-ops in an ordinary launch)
#define HODG_PDL 1
#endif
#ifndef HODG_PDL_MAX_ELEMS
#define HODG_PDL_MAX_ELEMS 200000
#endif
// the element bound, overridable at run time (env HODG_PDL_MAX_ELEMS; 0 = never)
inline int64_t hodg_pdl_max_elems() {
    static const int64_t v = [] {
        const char* s = getenv("HODG_PDL_MAX_ELEMS");
        return s ? int64_t(strtoll(s, nullptr, 10)) : int64_t(HODG_PDL_MAX_ELEMS);
    }();
    return v;
}
#ifndef HODG_EMINB
#define HODG_EMINB 0
#endif
// CTAs per SM the FP64 element kernel is register-budgeted for
// (P2 FP64: 4 CTAs -- 96 registers and, with 4 volume points per chunk and
// unpadded record rows, 56.9 KB of shared memory: 20 warps per SM instead of 15)
constexpr int EMINB = HODG_EMINB ? HODG_EMINB : (H > 1 ? 2 : (ORDER == 2 ? 4 : 3));
#ifndef HODG_U0_TMA_ORDER
#define HODG_U0_TMA_ORDER 0  // orders >= this fetch u0 by TMA after the volume phases (else: registers)
#endif
constexpr bool U0_TMA = ORDER >= HODG_U0_TMA_ORDER;  // CTAs per SM the FP64 element kernel is register-budgeted for
constexpr int XS = 15;                        // smem slot per (element, qp): 5 traces -> 15 contravariant fluxes
#ifndef HODG_QC2F
#define HODG_QC2F 5  // P2 mixed precision
#endif
#ifndef HODG_QC2
#define HODG_QC2 4
#endif
#ifndef HODG_QC3
#define HODG_QC3 6
#endif
// volume qps per chunk (bounds the X buffer; at P3 small enough for 4 CTAs/SM)
// volume points per chunk of the element kernel, per arithmetic type
template <typename T>
__host__ __device__ constexpr int qc() {
    return (NQV <= 8) ? NQV : (ORDER == 2 ? (sizeof(T) == 8 ? HODG_QC2 : HODG_QC2F) : HODG_QC3);
}

// padded per-face record of the face flux buffer: 5 x NQF values rounded up
// to 16 bytes so each face is one TMA bulk copy
template <typename T>
__host__ __device__ constexpr int hstride() {
    return int(((5 * NQF * sizeof(T) + 15) / 16) * 16 / sizeof(T));
}
// smem stride of the gathered face records: padded for the bank pattern,
// except at P2 where the unpadded rows let 4 FP64 element CTAs fit an SM
#ifndef HODG_HSS_NOPAD
#define HODG_HSS_NOPAD (ORDER == 2)
#endif
constexpr bool HSS_NOPAD = HODG_HSS_NOPAD;
template <typename T>
__host__ __device__ constexpr int hsmem() {
    // FP32: a stride that is a multiple of 32 words would put every element
    // of a warp on one bank; +4 words keeps 16-byte alignment (4-way at most)
    if (sizeof(T) == 4) return hstride<T>() % 32 == 0 ? hstride<T>() + 4 : hstride<T>();
    if (HSS_NOPAD) return hstride<T>();
    return (hstride<T>() % 4 == 2) ? hstride<T>() : hstride<T>() + 2;
}

// element-slot record block: the 4 face records of an element (5 x NQF
// values each, slot-major, unpadded) plus one pad value, so the stride is
// odd (conflict-free per-element smem access) and an E-element tile is a
// 16-byte multiple (one TMA bulk copy per tile)
// (warp-group kernel: even, so a 6-element group of FP32 blocks is a 16-byte
// multiple)
constexpr int HSE = 5 * NQF;
constexpr int EREC = WARP_ELEM ? 4 * HSE + 2 : 4 * HSE + 1;

__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~size_t(15); }
__host__ __device__ constexpr size_t cmax(size_t a, size_t b) { return a > b ? a : b; }

// compile-time loop: f(std::integral_constant<int, I>) for I in [0, N)
template <typename F, int... Is>
__device__ __forceinline__ void sfor_impl(F&& f, std::integer_sequence<int, Is...>) {
    (f(std::integral_constant<int, Is>{}), ...);
}
template <int N, typename F>
__device__ __forceinline__ void sfor(F&& f) {
    sfor_impl(f, std::make_integer_sequence<int, N>{});
}

// load n consecutive doubles starting at a 16-byte aligned address with
// 128-bit loads (conflict-free at the element kernel's row strides)
template <int N>
__device__ __forceinline__ void ld_row(const double* src, double (&dst)[N]) {
#pragma unroll
    for (int k = 0; k + 1 < N; k += 2) {
        const double2 p = *reinterpret_cast<const double2*>(src + k);
        dst[k] = p.x;
        dst[k + 1] = p.y;
    }
    if constexpr (N % 2 == 1) dst[N - 1] = src[N - 1];
}

// a face record's NQF values at offset `off` (parity known at compile
// time): 128-bit loads on the aligned pairs
template <int NQ, int START>
__device__ __forceinline__ void ld_rec(const double* rec, double (&dst)[NQ]) {
    if constexpr (START == 1) dst[0] = rec[0];
#pragma unroll
    for (int q = START; q + 1 < NQ; q += 2) {
        const double2 p = *reinterpret_cast<const double2*>(rec + q);
        dst[q] = p.x;
        dst[q + 1] = p.y;
    }
    if constexpr ((NQ - START) % 2 == 1) dst[NQ - 1] = rec[NQ - 1];
}

// exponent d of monomial i in the graded order (degree, then descending x,
// then descending y): the reference's `_EXPONENTS` order (hodg/basis.py:21) in 3D
__host__ __device__ constexpr int expt(int i, int d) {
    int k = 0, base = 0;
    while (base + (k + 1) * (k + 2) / 2 <= i) {
        base += (k + 1) * (k + 2) / 2;
        ++k;
    }
    int r = i - base, a = k;
    while (r >= k - a + 1) {
        r -= k - a + 1;
        --a;
    }
    const int b = k - a - r;
    return d == 0 ? a : (d == 1 ? b : k - a - b);
}

// R: element type of the state rows the face kernel reads -- the FP64 state,
// or (mixed precision) its FP32 shadow
// row buffers of the face kernel: 2 (the next tile's rows stream in during
// this tile's Riemann phase) or 1 (less shared memory: more CTAs per SM,
// the next tile's copies issued after the Riemann phase)
// (P3: one buffer at 5 CTAs per SM, 94 registers, measured 4.5% faster;
// P1 / P2: two buffers at 4 CTAs)
#ifndef HODG_FACE_NBUF
#define HODG_FACE_NBUF (ORDER == 3 ? 1 : 2)
#endif
constexpr int FNBUF = HODG_FACE_NBUF;
// state rows by TMA tile::gather4: four (face, side) rows per instruction
// (one per row otherwise); rows land in 128-byte-aligned groups of four.
// Off: faster (FP64 P2 face 0.489 -> 0.475 ms, mixed 0.334 -> 0.322 ms) and
// parity-green in isolation, but one GPU-suite ordering (the 2D, halo and
// multi-rank tests before the parity tests) hits an illegal-address fault in
// the P1 face launch with it, reproducibly, and never without it; the cause
// is not found, so the shipped default is the per-row
// bulk copy
#ifndef HODG_FACE_G4
#define HODG_FACE_G4 0
#endif
constexpr bool FG4 = HODG_FACE_G4 && !HODG_FACE_CPASYNC;
// phase-1 traces without per-qp branches or zero-initialised accumulators
// (1: except FP64 P3, where it measured 0.704 -> 0.750 ms; 2: everywhere)
#ifndef HODG_FACE_P1_FLAT
#define HODG_FACE_P1_FLAT 1
#endif
#ifndef HODG_G4_EXACT
#define HODG_G4_EXACT 0  // debug: the row map's extent = n_elems (ghost rows would read as zeros)
#endif
#ifndef HODG_G4_DEBUG
#define HODG_G4_DEBUG 0
#endif
#ifndef HODG_TM_FENCE
#define HODG_TM_FENCE 0
#endif
// FP32 contractions as packed f32x2 FMAs (FFMA2: two FMAs per issue slot)
#ifndef HODG_FFMA2
#define HODG_FFMA2 1
#endif
// FP32 Roe with the two sides in f32x2 lanes (roe_x2): measured off -- the
// packing moves and horizontal sums eat the saved slots (P2 face 0.296 vs
// 0.296 ms, P1 0.212 -> 0.217 ms)
#ifndef HODG_ROE_X2
#define HODG_ROE_X2 0
#endif
// phase-1 coefficient loads in pairs (one 16-byte / 8-byte shared load):
// measured off -- FP64 P2 face 0.462 vs 0.463 ms, mixed 0.297 -> 0.304 ms
#ifndef HODG_FACE_VEC
#define HODG_FACE_VEC 0
#endif
template <typename T>
__host__ __device__ constexpr bool face_p1_flat() {
    return HODG_FACE_P1_FLAT == 2 || (HODG_FACE_P1_FLAT == 1 && !(ORDER == 3 && sizeof(T) == 8));
}
template <typename R>
__host__ __device__ constexpr int g4_stride() {  // elements per group of four rows
    return int((4 * rstride<R>() * sizeof(R) + 127) / 128 * 128 / sizeof(R));
}
// smem offset (elements) of the row of (face, side) slot k = side * FT + lf
template <typename R>
__host__ __device__ constexpr int row_slot(int k) {
    return FG4 ? (k >> 2) * g4_stride<R>() + (k & 3) * rstride<R>() : k * rstride<R>();
}
__host__ __device__ constexpr size_t align128(size_t x) { return (x + 127) & ~size_t(127); }
template <typename T, typename R = double>
__host__ __device__ constexpr size_t face_smem_bytes() {
    return (FG4 ? align128(16 + 4 * FBS * sizeof(T)) : align16(16 + 4 * FBS * sizeof(T))) +
           FNBUF * (FG4 ? align128(cmax(size_t(row_slot<R>(2 * FT)) * sizeof(R), size_t(2 * FT) * NQF * 5 * sizeof(T)))
                        : align16(cmax(size_t(2 * FT) * rstride<R>() * sizeof(R),
                                       size_t(2 * FT) * NQF * 5 * sizeof(T))));
}

// element kernel shared memory carve-up
// element kernel shared memory carve-up.  The state tile lands in the record
// region and is read into registers before the records are fetched over it;
// the u0 tile, then the output tile, reuse the per-chunk X region, followed
// by the reduction slots.  Persistent CTAs (EPERSIST) double-buffer the
// geometry / face-id tiles and prefetch the next tile's inputs into the
// record region once the gather has consumed it.
#ifndef HODG_EPERSIST
#define HODG_EPERSIST 0
#endif
constexpr bool EPERSIST = HODG_EPERSIST && !WARP_ELEM && ORDER <= 2 && H == 1;
#ifndef HODG_RED_HT
#define HODG_RED_HT 1
#endif

// face-ordered records by TMA tile::gather4 (four records per instruction),
// in 128-byte-aligned groups of four.  1: FP64 (P0 / P1 / P2 element kernel
// 0.128 / 0.252 / 0.464 -> 0.109 / 0.240 / 0.444 ms at C1M); 2: also FP32,
// whose groups put a warp's record reads on few banks (P2 0.345 -> 0.388 ms).
// Off by default, as HODG_FACE_G4: with gather4 in the kernels the full GPU
// suite hit an illegal-address fault in 2 of 7 runs (never without it)
#ifndef HODG_ELEM_G4
#define HODG_ELEM_G4 0
#endif
template <typename T>
__host__ __device__ constexpr bool elem_g4() {
    return !(sizeof(T) == 4 ? HODG_ELEM_CPASYNC_F : HODG_ELEM_CPASYNC) &&
           (HODG_ELEM_G4 == 2 || (HODG_ELEM_G4 == 1 && sizeof(T) == 8));
}
// smem offset (elements) of face record r = s * E + e in the face-ordered tile
template <typename T>
__host__ __device__ constexpr int rec_slot(int r) {
    return elem_g4<T>() ? (r >> 2) * int(align128(4 * hstride<T>() * sizeof(T)) / sizeof(T)) + (r & 3) * hstride<T>()
                        : r * hsmem<T>();
}

template <typename T, bool ES>
struct ElemSmem {
    static constexpr int NGB = EPERSIST ? 2 : 1;
    static constexpr size_t bar = 0;                                         // in[2], records, u0 tile
    static constexpr size_t geo = 32;                                        // NGB x 16 x E doubles (tiled)
    static constexpr size_t fid = geo + size_t(NGB) * 16 * E * 8;            // NGB x 4 x E int32 (tiled)
    static constexpr size_t htile = !ES && elem_g4<T>() ? align128(fid + size_t(NGB) * 4 * E * 4)
                                                        : align16(fid + size_t(NGB) * 4 * E * 4);  // state tile, then the records
    static constexpr size_t hrec = ES ? size_t(E) * EREC * sizeof(T) : size_t(rec_slot<T>(4 * E)) * sizeof(T);
    static constexpr size_t sbytes = size_t(E) * RS * 8;
    static constexpr size_t hbytes = EPERSIST ? cmax(hrec, sbytes) : hrec;
    static constexpr size_t sx = align16(htile + hbytes);
    static constexpr size_t s32_bytes = sizeof(T) == 4 ? size_t(E) * RSF * 4 : 0;
    static constexpr size_t red_bytes = size_t(5 + 5 * H) * E * 8;
    // mixed precision: the reduction slots and the FP32 output tile reuse the
    // record region once the gather has consumed it (one barrier), so a CTA
    // is the records + max(state / output tile, X) only
    static constexpr bool rht =
        HODG_RED_HT && sizeof(T) == 4 && H == 1 && !EPERSIST && red_bytes + s32_bytes <= hbytes;
    static constexpr size_t red = rht ? htile : sx + sbytes;                 // (5 + 5H) x E doubles
    static constexpr size_t s32 = red + red_bytes;                           // mixed: FP32 output tile
    static constexpr size_t sx_bytes = rht ? cmax(sbytes, size_t(qc<T>()) * E * XS * sizeof(T))
                                           : cmax(sbytes + red_bytes + s32_bytes, size_t(qc<T>()) * E * XS * sizeof(T));
    static constexpr size_t total = sx + sx_bytes;
    // H > 1: the residual exchange of the mass solve reuses the record tile
    static_assert(H == 1 || hbytes >= size_t(5) * E * NB * 8, "solve exchange fits the record tile");
};

template <typename T, bool ES>
__host__ __device__ constexpr size_t elem_smem_bytes() {
    return ElemSmem<T, ES>::total;
}

// h (runtime, warp-uniform) -> compile-time constant
template <typename F>
__device__ __forceinline__ void hsel(int h, F&& f) {
    if constexpr (H == 1) {
        f(std::integral_constant<int, 0>{});
    } else if constexpr (H == 2) {
        if (h == 0) f(std::integral_constant<int, 0>{});
        else f(std::integral_constant<int, 1>{});
    } else {
        static_assert(H <= 2, "basis split of 1 or 2");
    }
}

// ---------------------------------------------------------------------------
// Face gather of one local face s: fa[i] = sum_q FG[s][q][i0 + i] h[q] for
// this thread's basis functions [i0, i0 + N).  On faces s = 1, 2, 3 the
// coordinate eta_{s-1} is -1/4 at every point (the face opposite vertex s of
// the reference tetrahedron has xi_{s-1} = 0), so the weighted trace of a
// monomial with exponent c > 0 in that coordinate is (-1/4)^c times the
// trace of the monomial without it: exactly, since the factor is a power of
// two (refelem.py builds the tables as products).  Only the c = 0 monomials
// are contracted (P2: 6 of 10, P3: 10 of 20); the rest are one scaling each
// and equal the direct contraction bit for bit.
#ifndef HODG_FOLD
#define HODG_FOLD 1
#endif
template <typename T, int S0, int I0, int N, int NQ>
__device__ __forceinline__ void face_moments(const T (&hq)[NQ], T (&fa)[N]) {
    constexpr int S = S0;
    constexpr bool FOLD = HODG_FOLD && !(HODG_FOLD == 2 && N != NB);  // 2: only without a basis split
    constexpr int d = S - 1;
    auto direct = [](auto i) {
        return !FOLD || S == 0 || expt(I0 + decltype(i)::value, d < 0 ? 0 : d) == 0;
    };
    // points outer, basis inner: consecutive table entries pair into 128-bit
    // constant loads (LDCU.128)
    sfor<N>([&](auto i) {
        if constexpr (direct(i)) fa[i] = T(0);
    });
    sfor<NQ>([&](auto q) {
        sfor<N>([&](auto i) {
            if constexpr (direct(i)) fa[i] += TAB(FG, T, (S * NQ + q) * NB + I0 + i) * hq[q];
        });
    });
    if constexpr (FOLD && S > 0) {
        sfor<N>([&](auto i) {
            constexpr int ig = I0 + i;
            constexpr int c = expt(ig, d);
            if constexpr (c > 0) {
                constexpr int base = mono_index(expt(ig, 0) - (d == 0 ? c : 0), expt(ig, 1) - (d == 1 ? c : 0),
                                                expt(ig, 2) - (d == 2 ? c : 0));
                static_assert(base >= I0 && base < I0 + N || N != NB, "full basis per thread holds the base");
                if constexpr (base >= I0 && base < I0 + N) {
                    constexpr double sc = c == 1 ? -0.25 : (c == 2 ? 0.0625 : -0.015625);
                    fa[i] = T(sc) * fa[base - I0];
                } else {
                    // basis split: the base function lives in the other part
                    T x = T(0);
                    sfor<NQ>([&](auto q) { x += TAB(FG, T, (S * NQ + q) * NB + ig) * hq[q]; });
                    fa[i] = x;  // (rare: only with H > 1)
                }
            }
        });
    }
}

// ---------------------------------------------------------------------------
// Face kernel: hodg/dg.py:240-351.  One CTA = FT faces.
//  phase 0: each (face, side) thread bulk-copies its element's state row
//           (TMA, cp.async.bulk) into shared memory;
//  phase 1: thread (face, side, qp-group) evaluates the side's traces at the
//           face quadrature points (reference-basis values of its local face
//           slot, staged in smem; coefficients reused across qps, basis values
//           across the 5 variables);
//  phase 2: thread (face, qp) closes boundary faces with the BC state and
//           evaluates the Roe / LLF flux, writing H[f][v][q] (padded record).
//  With ES the records go to the element-slot layout instead: each face's
//  record is stored in the blocks of both (owned) neighbours, so the element
//  kernel fetches a tile's records with one contiguous copy.
template <typename T, bool BND, bool ES, typename R = double>
__global__ void __launch_bounds__(FACE_THREADS, (sizeof(T) == 4 ? HODG_FACE_MINB_F : HODG_FACE_MINB) * 128 / FACE_THREADS)
    face_flux_kernel(const hodg_mesh_desc m, const R* __restrict__ state, T* __restrict__ hbuf,
                     uint32_t* __restrict__ err, int64_t f_begin, int64_t f_end,
                     const __grid_constant__ CUtensorMap rmap) {
    constexpr int HS = hstride<T>();
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);  // one per buffer
    T* fbt = reinterpret_cast<T*>(smem + 16);
    constexpr int RR = rstride<R>();
    R* rows0 = reinterpret_cast<R*>(smem + (FG4 ? align128(16 + 4 * FBS * sizeof(T)) : align16(16 + 4 * FBS * sizeof(T))));
    constexpr size_t BUF =
        (FG4 ? align128(cmax(size_t(row_slot<R>(2 * FT)) * sizeof(R), size_t(2 * FT) * NQF * 5 * sizeof(T)))
             : align16(cmax(size_t(2 * FT) * RR * sizeof(R), size_t(2 * FT) * NQF * 5 * sizeof(T)))) /
        sizeof(R);
    __shared__ double fn[2][FT][3];
    __shared__ int finf[2][FT];
    __shared__ int64_t fdst[2][FT][2];  // ES: record offsets of the left / right blocks (-1: none)

    const int t = threadIdx.x;
    const int side = t / (FT * NG);
    const int rem = t - side * FT * NG;
    const int lf = rem / NG;
    const int g = rem - lf * NG;
    if (t == 0) {
        mbar_init(bar, FACE_THREADS);
        mbar_init(bar + 1, FACE_THREADS);
        mbar_fence_init();
    }
    // stage the face trace table from its global-memory copy (coalesced; a
    // runtime-indexed __constant__ read would serialise across the warp)
    const T* fbg = sizeof(T) == 8 ? reinterpret_cast<const T*>(FBG_D) : reinterpret_cast<const T*>(FBG_F);
    for (int k = t; k < 4 * NQF * NB; k += FACE_THREADS) {
        const int s = k / (NQF * NB);
        fbt[s * FBS + (k - s * NQF * NB)] = fbg[k];
    }

    // per-tile metadata of this thread's (face, side): raw element id and
    // face info word (decoded only when consumed, so the loads issued for
    // the next tile stay in flight across this tile's work), and for the
    // (side 0, group 0) threads the right-element id and the normal
    struct Meta {
        int elem;
        int info;
        int right;
        double4 nrm;
    };
    const int ntiles = int((f_end - f_begin + FT - 1) / FT);
    auto load_meta = [&](int tile) {
        Meta mt{-1, 0, -1, make_double4(0, 0, 0, 0)};
        const int64_t f0 = f_begin + int64_t(tile) * FT;
        if (tile < ntiles && f0 + lf < f_end) {
            const int64_t f = f0 + lf;
            mt.elem = __ldg(m.fcells + 2 * f + side);
            mt.info = __ldg(m.finfo + f);
            if (side == 0 && g == 0) {
                mt.right = __ldg(m.fcells + 2 * f + 1);
                const double2 a = __ldg(reinterpret_cast<const double2*>(m.fnrm) + 2 * f);
                const double2 b = __ldg(reinterpret_cast<const double2*>(m.fnrm) + 2 * f + 1);
                mt.nrm = make_double4(a.x, a.y, b.x, b.y);
            }
        }
        return mt;
    };
    auto publish = [&](const Meta& mt, int buf) {
        if (side == 0 && g == 0) {
            finf[buf][lf] = ((mt.info >> 4) & 15) | (mt.right >= 0 ? 0x100 : 0);
            if constexpr (ES) {
                fdst[buf][lf][0] = mt.elem < m.n_elems ? int64_t(mt.elem) * EREC + (mt.info & 3) * HSE : -1;
                fdst[buf][lf][1] = (mt.right >= 0 && mt.right < m.n_elems)
                                       ? int64_t(mt.right) * EREC + ((mt.info >> 2) & 3) * HSE
                                       : -1;
            }
            fn[buf][lf][0] = mt.nrm.x;
            fn[buf][lf][1] = mt.nrm.y;
            fn[buf][lf][2] = mt.nrm.z;
        }
        R* row = rows0 + buf * BUF + row_slot<R>(side * FT + lf);
        if constexpr (FG4) {
            // faces lf .. lf+3 of this side sit NG lanes apart in the warp
            const int e1 = __shfl_down_sync(0xffffffffu, mt.elem, NG);
            const int e2 = __shfl_down_sync(0xffffffffu, mt.elem, 2 * NG);
            const int e3 = __shfl_down_sync(0xffffffffu, mt.elem, 3 * NG);
            if (g == 0 && (lf & 3) == 0) {
#if HODG_G4_DEBUG
                {
                    const int lim = int(2 * m.n_faces);  // (ghost rows sit past n_elems)
                    const bool bad_idx = mt.elem < -1 || mt.elem >= lim || e1 < -1 || e1 >= lim || e2 < -1 ||
                                         e2 >= lim || e3 < -1 || e3 >= lim;
                    const bool bad_dst = (smem_u32(row) & 127u) != 0;
                    const bool bad_map = (reinterpret_cast<uintptr_t>(&rmap) & 63u) != 0;
                    if (bad_idx || bad_dst || bad_map) {
                        printf("G4DBG blk %d side %d lf %d idx %d %d %d %d lim %d dst %u map %p f0 %lld fe %lld\n",
                               int(blockIdx.x), side, lf, mt.elem, e1, e2, e3, lim, smem_u32(row),
                               (const void*)&rmap, (long long)f_begin, (long long)f_end);
                        __trap();
                    }
                }
#endif
                mbar_arrive_expect_tx(bar + buf, 4 * RR * sizeof(R));
                tma_gather4(row, &rmap, mt.elem, e1, e2, e3, bar + buf);
            } else {
                mbar_arrive(bar + buf);
            }
            return;
        }
#if HODG_FACE_CPASYNC
        // the NG threads of this (face, side) copy the row in 16-byte
        // chunks, interleaved so each adjacent pair fills one 32-byte sector
        if (mt.elem >= 0) {
            const char* src = reinterpret_cast<const char*>(state + int64_t(mt.elem) * RR);
            char* dst = reinterpret_cast<char*>(row);
#pragma unroll
            for (int ch = g; ch < RR * int(sizeof(R)) / 16; ch += NG) cp_async16(dst + 16 * ch, src + 16 * ch);
            cp_async_arrive(bar + buf);
        } else {
            mbar_arrive(bar + buf);
        }
#else
        if (g == 0 && mt.elem >= 0) {
            mbar_arrive_expect_tx(bar + buf, RR * sizeof(R));
            bulk_g2s(row, state + int64_t(mt.elem) * RR, RR * sizeof(R), bar + buf);
        } else {
            mbar_arrive(bar + buf);
        }
#endif
    };

    int tile = blockIdx.x;
    Meta cur = load_meta(tile);
#if HODG_TM_FENCE
    if constexpr (FG4) {
        // make the TMA unit see this launch's row map (a descriptor cached
        // from an earlier launch at the same parameter address would be stale)
        asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(&rmap) : "memory");
    }
#endif
    __syncthreads();  // barrier init visible
    // programmatic dependent launch: the prologue above (barriers, face
    // table, first metadata) overlapped the previous kernel's tail; its state
    // rows and the record buffer it reads need it complete.  Dependents are
    // released only after this wait, so a kernel two launches ahead never
    // overlaps the one that produced its inputs.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    if (tile < ntiles) publish(cur, 0);
    const T gam = T(m.gamma);
    for (int it = 0; tile < ntiles; tile += gridDim.x, ++it) {
        const int buf = FNBUF == 2 ? (it & 1) : 0;
        const int64_t f0 = f_begin + int64_t(tile) * FT;
        const int nf = int(min(int64_t(FT), f_end - f0));
        const Meta nxt = load_meta(tile + gridDim.x);  // in flight during this tile
        mbar_wait(bar + buf, FNBUF == 2 ? ((it >> 1) & 1) : (it & 1));

        // phase 1: traces of this side at qps [g*QPT, g*QPT + QPT)
        const R* myrow = rows0 + buf * BUF + row_slot<R>(side * FT + lf);
        T tr[QPT][5];
        if constexpr (!face_p1_flat<T>()) {
#pragma unroll
            for (int qq = 0; qq < QPT; ++qq)
#pragma unroll
                for (int v = 0; v < 5; ++v) tr[qq][v] = T(0);
            if (cur.elem >= 0) {
                const int slot = side == 0 ? (cur.info & 3) : ((cur.info >> 2) & 3);
                const T* fb = fbt + slot * FBS;
#pragma unroll
                for (int i = 0; i < NB; ++i) {
                    T c[5];
#pragma unroll
                    for (int v = 0; v < 5; ++v) c[v] = T(myrow[v * NB + i]);
#pragma unroll
                    for (int qq = 0; qq < QPT; ++qq) {
                        const int q = g * QPT + qq;
                        if (NG * QPT == NQF || q < NQF) {
                            const T b = fb[q * NB + i];
#pragma unroll
                            for (int v = 0; v < 5; ++v) tr[qq][v] += b * c[v];
                        }
                    }
                }
            }
        } else if (FG4 || cur.elem >= 0) {
            // (gather4 zero-fills the rows of absent elements: no branch)
            const int slot = side == 0 ? (cur.info & 3) : ((cur.info >> 2) & 3);
            const T* fb = fbt + slot * FBS;
            // a group's qps past NQF repeat the last one (not stored): no
            // per-qp branch inside the basis loop
            int qo[QPT];
#pragma unroll
            for (int qq = 0; qq < QPT; ++qq) qo[qq] = min(g * QPT + qq, NQF - 1) * NB;
            if constexpr (sizeof(T) == 4 && HODG_FFMA2 && QPT >= 2) {
                // FP32: two qps per packed FFMA2 (sm_100 f32x2: the pair of
                // table values against the coefficient broadcast) -- per
                // lane the same FMUL / FFMA as the scalar loop
                constexpr int NP = QPT / 2;
                float2 t2[NP][5];
#pragma unroll
                for (int i = 0; i < NB; ++i) {
                    float c[5];
#pragma unroll
                    for (int v = 0; v < 5; ++v) c[v] = float(myrow[v * NB + i]);
#pragma unroll
                    for (int pp = 0; pp < NP; ++pp) {
                        const float2 b2 = make_float2(float(fb[qo[2 * pp] + i]), float(fb[qo[2 * pp + 1] + i]));
#pragma unroll
                        for (int v = 0; v < 5; ++v)
                            t2[pp][v] = i == 0 ? __fmul2_rn(b2, make_float2(c[v], c[v]))
                                               : __ffma2_rn(b2, make_float2(c[v], c[v]), t2[pp][v]);
                    }
                    if constexpr (QPT % 2 == 1) {
                        const float b = float(fb[qo[QPT - 1] + i]);
#pragma unroll
                        for (int v = 0; v < 5; ++v)
                            tr[QPT - 1][v] = i == 0 ? T(b * c[v]) : T(fmaf(b, c[v], float(tr[QPT - 1][v])));
                    }
                }
#pragma unroll
                for (int pp = 0; pp < NP; ++pp)
#pragma unroll
                    for (int v = 0; v < 5; ++v) {
                        tr[2 * pp][v] = T(t2[pp][v].x);
                        tr[2 * pp + 1][v] = T(t2[pp][v].y);
                    }
            } else if constexpr (HODG_FACE_VEC && NB % 2 == 0) {
                // coefficient pairs (i, i+1) by one 16-byte (FP32: 8-byte)
                // shared load; the sums keep the basis order
#pragma unroll
                for (int i = 0; i < NB; i += 2) {
                    T c0[5], c1[5];
#pragma unroll
                    for (int v = 0; v < 5; ++v) {
                        if constexpr (sizeof(R) == 8) {
                            const double2 d = *reinterpret_cast<const double2*>(myrow + v * NB + i);
                            c0[v] = T(d.x);
                            c1[v] = T(d.y);
                        } else {
                            const float2 d = *reinterpret_cast<const float2*>(myrow + v * NB + i);
                            c0[v] = T(d.x);
                            c1[v] = T(d.y);
                        }
                    }
#pragma unroll
                    for (int qq = 0; qq < QPT; ++qq) {
                        const T b0 = fb[qo[qq] + i], b1 = fb[qo[qq] + i + 1];
#pragma unroll
                        for (int v = 0; v < 5; ++v) {
                            const T x = i == 0 ? b0 * c0[v] : tr[qq][v] + b0 * c0[v];
                            tr[qq][v] = x + b1 * c1[v];
                        }
                    }
                }
            } else {
#pragma unroll
                for (int i = 0; i < NB; ++i) {
                    T c[5];
#pragma unroll
                    for (int v = 0; v < 5; ++v) c[v] = T(myrow[v * NB + i]);
#pragma unroll
                    for (int qq = 0; qq < QPT; ++qq) {
                        const T b = fb[qo[qq] + i];
#pragma unroll
                        for (int v = 0; v < 5; ++v) tr[qq][v] = i == 0 ? b * c[v] : tr[qq][v] + b * c[v];
                    }
                }
            }
        } else {
#pragma unroll
            for (int qq = 0; qq < QPT; ++qq)
#pragma unroll
                for (int v = 0; v < 5; ++v) tr[qq][v] = T(0);
        }
        __syncthreads();  // rows[buf] consumed; previous tile's phase 2 done everywhere
        T* trs = reinterpret_cast<T*>(rows0 + buf * BUF);
        if (lf < nf) {
#pragma unroll
            for (int qq = 0; qq < QPT; ++qq) {
                const int q = g * QPT + qq;
                if (NG * QPT == NQF || q < NQF) {
#pragma unroll
                    for (int v = 0; v < 5; ++v) trs[(size_t(side * FT + lf) * NQF + q) * 5 + v] = tr[qq][v];
                }
            }
        }
        // next tile: its rows stream into the other buffer during phase 2
        if (FNBUF == 2 && tile + gridDim.x < ntiles) publish(nxt, buf ^ 1);
        __syncthreads();

        // phase 2: Riemann flux at each (face, qp); two pairs per thread per
        // iteration so their (straight-line) Roe evaluations interleave
        const int npairs = nf * NQF;
        for (int p0 = t; p0 < npairs; p0 += RP * FACE_THREADS) {
            T qL[RP][5], qR[RP][5], h[RP][5], n[RP][3];
            bool ok[RP];
            int64_t fid[RP];
            int qv[RP];
            int lfv[RP];
#pragma unroll
            for (int k = 0; k < RP; ++k) {
                const int p = min(p0 + k * FACE_THREADS, npairs - 1);
                const int lfp = p / NQF;
                const int q = p - lfp * NQF;
                fid[k] = f0 + lfp;
                qv[k] = q;
                lfv[k] = lfp;
                const int info = finf[buf][lfp];
#pragma unroll
                for (int d = 0; d < 3; ++d) n[k][d] = T(fn[buf][lfp][d]);
#pragma unroll
                for (int v = 0; v < 5; ++v) qL[k][v] = trs[(size_t(lfp) * NQF + q) * 5 + v];
                ok[k] = true;
                if (!BND || (info & 0x100)) {
#pragma unroll
                    for (int v = 0; v < 5; ++v) qR[k][v] = trs[(size_t(FT + lfp) * NQF + q) * 5 + v];
                } else if constexpr (BND) {
                    T u, vv, w;
                    if (!(qL[k][0] > T(0)) || !(prim(qL[k], gam, u, vv, w) > T(0))) {
                        ok[k] = false;
#pragma unroll
                        for (int v = 0; v < 5; ++v) qR[k][v] = qL[k][v];
                    } else {
                        const T qf[5] = {T(m.qinf[0]), T(m.qinf[1]), T(m.qinf[2]), T(m.qinf[3]), T(m.qinf[4])};
                        bstate(info & 15, qL[k], n[k], qf, gam, qR[k]);
                    }
                }
            }
            if (m.flux_kind == HODG_FLUX_LLF) {
                for (int k = 0; k < RP; ++k) ok[k] = ok[k] && llf(qL[k], qR[k], n[k], gam, h[k]);
            } else {
                bool r[RP];
#pragma unroll
                for (int k = 0; k < RP; ++k) {
                    if constexpr (sizeof(T) == 4 && HODG_ROE_X2)
                        r[k] = roe_x2(qL[k], qR[k], n[k], gam, h[k]);
                    else
                        r[k] = roe(qL[k], qR[k], n[k], gam, h[k]);
                }
#pragma unroll
                for (int k = 0; k < RP; ++k) ok[k] = ok[k] && r[k];
            }
#pragma unroll
            for (int k = 0; k < RP; ++k) {
                if (k >= 1 && p0 + k * FACE_THREADS >= npairs) break;
                if (!ok[k]) {
                    flag(err, 0, uint32_t(fid[k]));
#pragma unroll
                    for (int v = 0; v < 5; ++v) h[k][v] = T(0);
                }
                if constexpr (ES) {
                    const int64_t dl = fdst[buf][lfv[k]][0], dr = fdst[buf][lfv[k]][1];
                    if (dl >= 0) {
#pragma unroll
                        for (int v = 0; v < 5; ++v) hbuf[dl + v * NQF + qv[k]] = h[k][v];
                    }
                    if (dr >= 0) {
#pragma unroll
                        for (int v = 0; v < 5; ++v) hbuf[dr + v * NQF + qv[k]] = h[k][v];
                    }
                } else {
#pragma unroll
                    for (int v = 0; v < 5; ++v) hbuf[fid[k] * HS + v * NQF + qv[k]] = h[k][v];
                }
            }
        }
        if constexpr (FNBUF == 1) {
            // single buffer: the traces and this tile's metadata are consumed
            __syncthreads();
            if (tile + gridDim.x < ntiles) publish(nxt, 0);
        }
        cur = nxt;
    }
}

// ---------------------------------------------------------------------------
// Element kernel: hodg/dg.py:353-460 fused with the RK stage update
// (hodg/timestepping.py:165-180) and the next step's CFL dt
// (hodg/timestepping.py:105-134).  One CTA = E elements, thread (v, e).
//  phase 0: TMA bulk copies of the state / geometry / face-id tiles, then
//           one bulk copy per (element, face) of the face flux records --
//           in flight while the volume integral runs;
//  per chunk of QC volume points:
//    phase A: thread (v, e): traces of variable v (coefficients in registers);
//    phase B: thread (e, q): Euler flux, contravariant flux J^-1 F;
//    phase C: thread (v, e): volume integral (weighted derivative tables);
//  gather: thread (v, e): the four face fluxes against the face tables,
//  then the reference mass solve (FP64), RK combination, dt / norm epilogues.
// Geometry tiles are field-major ([tile][field][E]) so every smem access in
// the hot phases is unit-stride across the warp.
// ES: the records are in the element-slot layout -- one bulk copy of the
// tile's record blocks, issued with the state tile, no per-face gather.
// element kernel: L2 prefetch distance in tiles (0: off)
#ifndef HODG_EPF_DIST
#define HODG_EPF_DIST 0
#endif
constexpr int EPF_DIST = HODG_EPF_DIST;
#ifndef HODG_MP_FACE_F32
// mixed: face terms of the element residual accumulated in FP32 (as the
// volume term), one conversion for the FP64 solve -- P1 / P3 element kernel
// 0.192 / 0.552 -> 0.181 / 0.534 ms, P2 0.335 -> 0.340 ms.  Off: the
// reference's float32 rhs_pass adds each face term into its FP64 scratch
// (SURVEY.md appendix A), which the default keeps
#define HODG_MP_FACE_F32 0
#endif
#ifndef HODG_EMINB_F
#define HODG_EMINB_F 6  // mixed-precision element kernel at P0-P2 (64 registers; RED / FP32 tile in the record region)
#endif
template <typename T, bool ES>
__global__ void __launch_bounds__(ETHREADS, sizeof(T) == 4 ? (H > 1 ? 2 : HODG_EMINB_F) : EMINB)
    elem_stage_kernel(const hodg_mesh_desc m, const T* __restrict__ hbuf, const hodg_stage_args a,
                      uint32_t* __restrict__ err, const __grid_constant__ CUtensorMap hmap) {
    using L = ElemSmem<T, ES>;
    constexpr int HS = hstride<T>();
    constexpr int HSS = hsmem<T>();
    constexpr bool ECPA = sizeof(T) == 4 ? HODG_ELEM_CPASYNC_F : HODG_ELEM_CPASYNC;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::bar);  // [0, 1] inputs per buffer, [2] records, [3] u0
    T* HT = reinterpret_cast<T*>(smem + L::htile);
    // the state tile: in the record region when persistent (the next tile's
    // prefetch lands there), else in the X region, so the element-slot
    // records can be fetched at once, alongside it
    double* SIN = reinterpret_cast<double*>(smem + (EPERSIST ? L::htile : L::sx));
    double* Z = reinterpret_cast<double*>(smem + L::htile);      // H > 1: residual exchange (after the gather)
    double* S = reinterpret_cast<double*>(smem + L::sx);         // u0 tile, then the output tile
    T* X = reinterpret_cast<T*>(smem + L::sx);                   // per-chunk trace / flux slots
    // [0, 5E): norm terms; [5E + 5E h, 10E + 5E h): cell-mean partials of basis part h
    double* RED = reinterpret_cast<double*>(smem + L::red);
    float* S32 = reinterpret_cast<float*>(smem + L::s32);  // mixed: FP32 shadow of the output tile
    const bool shadow = sizeof(T) == 4 && a.out32 != nullptr;
    const int t = threadIdx.x;
    const int64_t ntiles = (m.n_elems + E - 1) / E;
    // thread (v, h, e): e fastest, so h is warp-uniform (E >= 32 when H > 1)
    const int e = t % E;
    const int h = (t / E) % H;
    const int v = t / (E * H);
    const int jb = h * NH;  // first basis function of this thread's part
    const bool need_u0 = a.combine == 1 || (a.combine == 0 && a.a != 0.0);
    const bool need_mean = a.combine >= 0 && (a.dt_next || a.dt_vec_out);
    const T gam = T(m.gamma);

    auto issue_inputs = [&](int64_t tl, int gb) {  // thread 0
        const int nn = int(min(int64_t(E), m.n_elems - tl * E));
        const uint32_t bs = uint32_t(nn) * RS * 8;
        mbar_arrive_expect_tx(bar + gb, bs + 16 * E * 8 + 4 * E * 4);
        bulk_g2s(SIN, a.us + tl * E * RS, bs, bar + gb);
        bulk_g2s(reinterpret_cast<double*>(smem + L::geo) + gb * 16 * E, m.egeo + tl * 16 * E, 16 * E * 8, bar + gb);
        bulk_g2s(reinterpret_cast<int32_t*>(smem + L::fid) + gb * 4 * E, m.efaces + tl * 4 * E, 4 * E * 4,
                 bar + gb);
    };
    int64_t tile = blockIdx.x;
    if (t == 0) {
        if (a.dt_reset && blockIdx.x == 0) *a.dt_reset = 0x7FF0000000000000ull;
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        mbar_init(bar + 2, ES ? 1 : (ECPA ? ETHREADS : 4 * E));
        mbar_init(bar + 3, 1);
        mbar_fence_init();
        if (tile < ntiles) issue_inputs(tile, 0);  // the stage state: two launches back
        if constexpr (EPF_DIST > 0) {
            // warm L2 with the inputs of the tile a CTA will start about one
            // wave later, so its first TMA wait is an L2 round trip
            const int64_t pt = tile + EPF_DIST;
            if (!EPERSIST && pt < ntiles) {
                const int nn = int(min(int64_t(E), m.n_elems - pt * E));
                bulk_prefetch_l2(a.us + pt * E * RS, uint32_t(nn) * RS * 8);
                bulk_prefetch_l2(m.egeo + pt * 16 * E, 16 * E * 8);
                if (need_u0 && a.u0 != a.us) bulk_prefetch_l2(a.u0 + pt * E * RS, uint32_t(nn) * RS * 8);
            }
        }
    }
    // programmatic dependent launch: everything above overlapped the face
    // kernel's tail; records, and the in-place output, need it complete
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if constexpr (ES && !EPERSIST) {
        // element-slot records: one bulk copy, in flight with the state tile
        if (t == 0 && tile < ntiles) {
            const int64_t e0 = tile * E;
            const int ne = int(min(int64_t(E), m.n_elems - e0));
            const uint32_t hb = uint32_t(align16(size_t(ne) * EREC * sizeof(T)));
            mbar_arrive_expect_tx(bar + 2, hb);
            bulk_g2s(HT, hbuf + e0 * EREC, hb, bar + 2);
        }
    }
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;");

    for (int it = 0; tile < ntiles; tile += gridDim.x, ++it) {
        const int gbuf = EPERSIST ? (it & 1) : 0;
        const double* G = reinterpret_cast<const double*>(smem + L::geo) + gbuf * 16 * E;
        const int32_t* FI = reinterpret_cast<const int32_t*>(smem + L::fid) + gbuf * 4 * E;
        const int64_t e0 = tile * E;
        const int ne = int(min(int64_t(E), m.n_elems - e0));
        const int64_t gid = e0 + e;
        const bool live = e < ne;
        mbar_wait(bar + gbuf, EPERSIST ? ((it >> 1) & 1) : (it & 1));

        double c[NH];
        double u0r[!U0_TMA ? NH : 1];
        if (live) {
            if constexpr (H == 1 && (NB % 2) == 0) {
                ld_row(SIN + e * RS + v * NB, c);  // rows 16-byte aligned when NB is even
            } else {
#pragma unroll
                for (int i = 0; i < NH; ++i) c[i] = SIN[e * RS + v * NB + jb + i];
            }
            if constexpr (!U0_TMA) {
                if (need_u0) {
                    if constexpr (H == 1 && (NB % 2) == 0) {
                        ld_row(a.u0 + gid * RS + v * NB, u0r);
                    } else {
#pragma unroll
                        for (int i = 0; i < NH; ++i) u0r[i] = a.u0[gid * RS + v * NB + jb + i];
                    }
                }
            }
        }
        __syncthreads();  // state tile consumed (persistent: the region receives the records)

        // face flux records, in flight during the volume integral
        if constexpr (ES && !EPERSIST) {
            // issued at kernel start, with the state tile
        } else if constexpr (ES) {
            if (t == 0 && ne > 0) {
                const uint32_t hb = uint32_t(align16(size_t(ne) * EREC * sizeof(T)));
                fence_proxy_async();
                mbar_arrive_expect_tx(bar + 2, hb);
                bulk_g2s(HT, hbuf + e0 * EREC, hb, bar + 2);
            } else if (t == 0) {
                mbar_arrive(bar + 2);
            }
        } else if constexpr (ECPA) {
            // 16-byte cp.async chunks: thread (row rr, chunk k) of RPR rows
            // per round copies chunk k of records rr, rr + RPR, ... (the
            // division is done once); every thread arrives once when its
            // copies land
            constexpr int NC = int(HS * sizeof(T) / 16);
            constexpr int RPR = ETHREADS / NC;
            constexpr int NR = (4 * E + RPR - 1) / RPR;
            if (t < RPR * NC) {
                const int rr = t / NC;
                const int k = t - rr * NC;
                const char* src = reinterpret_cast<const char*>(hbuf) + 16 * k;
                char* dst = reinterpret_cast<char*>(HT) + 16 * k;
#pragma unroll
                for (int j = 0; j < NR; ++j) {
                    const int r = rr + j * RPR;
                    if ((NR * RPR == 4 * E || r < 4 * E) && r % E < ne)
                        cp_async16(dst + size_t(r) * HSS * sizeof(T), src + int64_t(FI[r]) * (HS * sizeof(T)));
                }
            }
            cp_async_arrive(bar + 2);
        } else {
            if constexpr (elem_g4<T>()) {
                // thread (s, e), e % 4 == 0, gathers faces FI[s][e .. e+3]
                // (rows past the tile's end: index -1, zero-filled)
                if (t < 4 * E) {
                    if ((t & 3) == 0) {
                        const int4 f4 = *reinterpret_cast<const int4*>(FI + t);
                        const int eb = t % E;
                        fence_proxy_async();
                        mbar_arrive_expect_tx(bar + 2, 4 * HS * sizeof(T));
                        tma_gather4(HT + rec_slot<T>(t), &hmap, eb < ne ? f4.x : -1, eb + 1 < ne ? f4.y : -1,
                                    eb + 2 < ne ? f4.z : -1, eb + 3 < ne ? f4.w : -1, bar + 2);
                    } else {
                        mbar_arrive(bar + 2);
                    }
                }
            } else if (t < 4 * E) {
                // thread (s, e) for t < 4E fetches face FI[s][e]
                if (t % E < ne) {
                    fence_proxy_async();
                    mbar_arrive_expect_tx(bar + 2, HS * sizeof(T));
                    bulk_g2s(HT + size_t(t) * HSS, hbuf + int64_t(FI[t]) * HS, HS * sizeof(T), bar + 2);
                } else {
                    mbar_arrive(bar + 2);
                }
            }
        }

        T acc[NH];
#pragma unroll
        for (int i = 0; i < NH; ++i) acc[i] = T(0);
        T mom[MOMENTS ? NBL : 1][3];
#pragma unroll
        for (int j = 0; j < (MOMENTS ? NBL : 1); ++j) mom[j][0] = mom[j][1] = mom[j][2] = T(0);
        T ji[H == 1 ? 9 : 1];
        if constexpr (H == 1) {
#pragma unroll
            for (int k = 0; k < 9; ++k) ji[k] = T(G[k * E + e]);
        }
        constexpr int QC = qc<T>();
        constexpr int NCH = (NQV + QC - 1) / QC;
        sfor<NCH>([&](auto ch) {
            constexpr int q0 = ch * QC;
            constexpr int nq = (NQV - q0) < QC ? (NQV - q0) : QC;
            // phase A: traces of variable v (H > 1: partial sums of this part,
            // added in phase B in part order)
            if (live) {
                hsel(h, [&](auto hc) {
                    sfor<nq>([&](auto qq) {
                        T u = T(0);
                        sfor<NH>([&](auto i) { u += TAB(VB, T, (q0 + qq) * NB + hc * NH + i) * T(c[i]); });
                        X[(qq * E + e) * XS + hc * 5 + v] = u;
                    });
                });
            }
            __syncthreads();
            // phase B: thread (e, q): Euler flux (and J^-1 F when H > 1)
            for (int p = t; p < nq * E; p += ETHREADS) {
                const int qq = p / E;
                const int ee = p - qq * E;
                if (ee >= ne) continue;
                T* sl = X + (qq * E + ee) * XS;
                T U[5];
#pragma unroll
                for (int k = 0; k < 5; ++k) U[k] = sl[k];
                if constexpr (H > 1) {
#pragma unroll
                    for (int hh = 1; hh < H; ++hh)
#pragma unroll
                        for (int k = 0; k < 5; ++k) U[k] += sl[hh * 5 + k];
                }
                T u, vv, w;
                const T pr = (U[0] > T(0)) ? prim(U, gam, u, vv, w) : T(-1);
                if (!(pr > T(0))) {
                    flag(err, 1, uint32_t(e0 + ee));
#pragma unroll
                    for (int k = 0; k < XS; ++k) sl[k] = T(0);
                    continue;
                }
                // physical flux F[d][var]
                const T Hs = U[4] + pr;
                T F[15] = {U[1], U[1] * u + pr, U[1] * vv, U[1] * w, Hs * u,
                           U[2], U[2] * u, U[2] * vv + pr, U[2] * w, Hs * vv,
                           U[3], U[3] * u, U[3] * vv, U[3] * w + pr, Hs * w};
                if constexpr (H == 1) {
                    // the reference-frame map J^-1 is applied per variable later
#pragma unroll
                    for (int k = 0; k < 15; ++k) sl[k] = F[k];
                } else {
                    // H > 1: J^-1 F here (phase C threads hold no J^-1)
                    T jj[9];
#pragma unroll
                    for (int k = 0; k < 9; ++k) jj[k] = T(G[k * E + ee]);
#pragma unroll
                    for (int d = 0; d < 3; ++d)
#pragma unroll
                        for (int var = 0; var < 5; ++var)
                            sl[d * 5 + var] =
                                jj[3 * d] * F[var] + jj[3 * d + 1] * F[5 + var] + jj[3 * d + 2] * F[10 + var];
                }
            }
            __syncthreads();
            // phase C (volume): contravariant flux of variable v against the
            // weighted derivative table, this part's basis functions (MOMENTS:
            // the physical flux of variable v against the weighted lower
            // monomials; J^-1 and the derivative identity after the last chunk)
            if constexpr (MOMENTS) {
                if (live) {
                    sfor<nq>([&](auto qq) {
                        const T* sl = X + (qq * E + e) * XS;
                        const T fx = sl[v], fy = sl[5 + v], fz = sl[10 + v];
                        sfor<NBL>([&](auto j) {
                            const T wm = TAB(WV, T, (q0 + qq) * NB + j);
                            if constexpr (sizeof(T) == 4 && HODG_FFMA2) {
                                // (x, y) as one FFMA2 with the weight broadcast
                                const float2 m2 = __ffma2_rn(make_float2(fx, fy), make_float2(wm, wm),
                                                             make_float2(mom[j][0], mom[j][1]));
                                mom[j][0] = m2.x;
                                mom[j][1] = m2.y;
                            } else {
                                mom[j][0] += wm * fx;
                                mom[j][1] += wm * fy;
                            }
                            mom[j][2] += wm * fz;
                        });
                    });
                }
            } else if (live) {
                hsel(h, [&](auto hc) {
                    sfor<nq>([&](auto qq) {
                        const T* sl = X + (qq * E + e) * XS;
                        T fd[3];
                        if constexpr (H == 1) {
                            const T fx = sl[v], fy = sl[5 + v], fz = sl[10 + v];
                            fd[0] = ji[0] * fx + ji[1] * fy + ji[2] * fz;
                            fd[1] = ji[3] * fx + ji[4] * fy + ji[5] * fz;
                            fd[2] = ji[6] * fx + ji[7] * fy + ji[8] * fz;
                        } else {
                            fd[0] = sl[v];
                            fd[1] = sl[5 + v];
                            fd[2] = sl[10 + v];
                        }
                        sfor<NH>([&](auto i) {
                            constexpr int ig = hc * NH + i;
                            sfor<3>([&](auto d) {
                                if constexpr (expt(ig, d) > 0)
                                    acc[i] += TAB(VD, T, ((q0 + qq) * NB + ig) * 3 + d) * fd[d];
                            });
                        });
                    });
                });
            }
            __syncthreads();
        });
        if constexpr (MOMENTS) {
            // sum_q VD[q][i][d] (J^-1 F)_d = sum_d alpha_{i,d} sum_k Jinv[d][k] MOM[i - e_d][k]
            T mj[NBL][3];
#pragma unroll
            for (int j = 0; j < NBL; ++j)
#pragma unroll
                for (int d = 0; d < 3; ++d)
                    mj[j][d] = ji[3 * d] * mom[j][0] + ji[3 * d + 1] * mom[j][1] + ji[3 * d + 2] * mom[j][2];
            sfor<NB>([&](auto i) {
                T sum = T(0);
                sfor<3>([&](auto d) {
                    constexpr int al = expt(i, d);
                    if constexpr (al > 0) {
                        constexpr int lo =
                            mono_index(expt(i, 0) - (d == 0), expt(i, 1) - (d == 1), expt(i, 2) - (d == 2));
                        sum += T(al) * mj[lo][d];
                    }
                });
                acc[i] = sum;
            });
        }

        // the u0 tile is not held in registers through the volume phases:
        // one TMA copy into the freed X region, in flight during the gather
        // and the solve (each thread later reads, then overwrites with its
        // output, only its own entries)
        if constexpr (U0_TMA) {
            if (need_u0 && t == 0 && ne > 0) {
                const uint32_t bs = uint32_t(ne) * RS * 8;
                fence_proxy_async();
                mbar_arrive_expect_tx(bar + 3, bs);
                bulk_g2s(S, a.u0 + e0 * RS, bs, bar + 3);
            }
        }
        // face gather, mass solve, RK update
        mbar_wait(bar + 2, it & 1);
        double accd[NH];
        if (live) {
            // the four face terms are added in FP64 (the reference's float32
            // rhs_pass adds its FP32 products into an FP64 scratch);
            // HODG_MP_FACE_F32 sums them in FP32 first
#pragma unroll
            for (int i = 0; i < NH; ++i) accd[i] = double(acc[i]);
            hsel(h, [&](auto hc) {
                sfor<4>([&](auto s) {
                    const T* hrec =
                        ES ? HT + size_t(e) * EREC + s * HSE + v * NQF : HT + rec_slot<T>(s * E + e) + v * NQF;
                    T hq[NQF];
                    if constexpr (ES) {
#pragma unroll
                        for (int q = 0; q < NQF; ++q) hq[q] = hrec[q];
                    } else if constexpr (sizeof(T) == 8) {
                        // record rows are 16-byte aligned: 128-bit loads on aligned pairs
                        if ((v * NQF) & 1) ld_rec<NQF, 1>(hrec, hq);
                        else ld_rec<NQF, 0>(hrec, hq);
                    } else {
#pragma unroll
                        for (int q = 0; q < NQF; ++q) hq[q] = hrec[q];
                    }
                    T fa[NH];
                    face_moments<T, s, hc * NH, NH>(hq, fa);
                    const double fc = G[(9 + s) * E + e];
                    if constexpr (sizeof(T) == 8 || !HODG_MP_FACE_F32) {
#pragma unroll
                        for (int i = 0; i < NH; ++i) accd[i] -= fc * double(fa[i]);
                    } else {
                        const T fcf = T(fc);
#pragma unroll
                        for (int i = 0; i < NH; ++i) acc[i] -= fcf * fa[i];
                    }
                });
            });
            if constexpr (sizeof(T) == 4 && HODG_MP_FACE_F32) {
#pragma unroll
                for (int i = 0; i < NH; ++i) accd[i] = double(acc[i]);
            }
        }
        double full[H == 1 ? 1 : NB];
        if constexpr (H > 1) {
            // assemble the (v, e) residual vector of all parts (records consumed)
            __syncthreads();
            if (live) {
#pragma unroll
                for (int i = 0; i < NH; ++i) Z[(v * E + e) * NB + jb + i] = accd[i];
            }
            __syncthreads();
            if (live) {
#pragma unroll
                for (int k = 0; k < NB; ++k) full[k] = Z[(v * E + e) * NB + k];
            }
        }
        if constexpr (L::rht) __syncthreads();  // records consumed: the region takes RED / the FP32 tile
        if constexpr (EPERSIST) {
            // the records are consumed: the next tile's inputs stream into the
            // region during this tile's solve and epilogue
            __syncthreads();
            if (t == 0 && tile + gridDim.x < ntiles) {
                fence_proxy_async();
                issue_inputs(tile + gridDim.x, gbuf ^ 1);
            }
        }
        if (live) {
            double r[NH];
            hsel(h, [&](auto hc) {
                sfor<NH>([&](auto j) {
                    double z = 0.0;
                    if constexpr (H == 1) {
                        sfor<NB>([&](auto k) { z += MINV_T[j * NB + k] * accd[k]; });
                    } else {
                        sfor<NB>([&](auto k) { z += MINV_T[(hc * NH + j) * NB + k] * full[k]; });
                    }
                    r[j] = z;
                });
            });
            if (a.res) {
#pragma unroll
                for (int j = 0; j < NH; ++j) a.res[gid * RS + v * NB + jb + j] = r[j];
            }
            if (a.norm_partial && h == 0) RED[v * E + e] = G[14 * E + e] * r[0] * r[0];
            if (a.combine >= 0) {
                if constexpr (U0_TMA) {
                    if (need_u0) mbar_wait(bar + 3, it & 1);
                }
                const double dt = a.dt_is_vector ? a.dt[gid] : a.dt[0];
                double mean = 0.0;
                double outr[NH];
                hsel(h, [&](auto hc) {
                    sfor<NH>([&](auto j) {
                        double u0j = 0.0;
                        if (need_u0) {
                            if constexpr (!U0_TMA) u0j = u0r[j];
                            else u0j = S[e * RS + v * NB + hc * NH + j];  // u0 tile (TMA, above)
                        }
                        double o;
                        if (a.combine == 1) {
                            o = 0.5 * ((u0j + c[j]) + dt * r[j]);
                        } else {
                            o = a.b * (c[j] + dt * r[j]);
                            if (a.a != 0.0) o = a.a * u0j + o;
                        }
                        outr[j] = o;
                        if (need_mean) mean += MEAN_T[hc * NH + j] * o;  // (the dt epilogue's cell mean)
                    });
                });
                if constexpr (H == 1 && (NB % 2) == 0) {
#pragma unroll
                    for (int j = 0; j < NB; j += 2)
                        *reinterpret_cast<double2*>(S + e * RS + v * NB + j) = make_double2(outr[j], outr[j + 1]);
                } else {
#pragma unroll
                    for (int j = 0; j < NH; ++j) S[e * RS + v * NB + jb + j] = outr[j];
                }
                if constexpr (sizeof(T) == 4) {
                    if (shadow) {
#pragma unroll
                        for (int j = 0; j < NH; ++j) S32[e * RSF + v * NB + jb + j] = float(outr[j]);
                    }
                }
                if (need_mean) RED[5 * E + h * 5 * E + v * E + e] = mean;
            }
        }
        fence_proxy_async();
        __syncthreads();
        if (t == 0 && a.combine >= 0 && ne > 0) {
            bulk_s2g(a.out + e0 * RS, S, uint32_t(ne) * RS * 8);
            if (shadow) bulk_s2g(a.out32 + e0 * RSF, S32, uint32_t(ne) * RSF * 4);
        }
        // epilogues without a trailing barrier: fixed-order shuffle trees over
        // the (variable, element) pairs held by threads t < 5E (vn = t / E)
        const int lane = t & 31;
        const int vn = t / E;
        if (a.norm_partial && t < 5 * E) {
            // partial sum over the tile of vol * res_0^2 per variable; warp w
            // holds variable (32 w) / E (E >= 32) or two variables (E == 16)
            constexpr int W = E < 32 ? E : 32;
            double x = (e < ne) ? RED[vn * E + e] : 0.0;
#pragma unroll
            for (int o = W / 2; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            if (E <= 32) {
                if ((lane % W) == 0) a.norm_partial[tile * 5 + vn] = x;
            } else {  // E == 64: two warps per variable, combined in a fixed order
                __shared__ double half2[10];
                if (lane == 0) half2[(t / 32)] = x;
                __syncwarp();
                asm volatile("bar.sync 1, %0;" ::"r"(5 * E));  // the 5E threads of this epilogue
                if (t < 5) a.norm_partial[tile * 5 + t] = half2[2 * t] + half2[2 * t + 1];
                asm volatile("bar.sync 1, %0;" ::"r"(5 * E));  // half2 read before the next tile
            }
        }
        if (a.combine >= 0 && (a.dt_next || a.dt_vec_out) && t < E) {
            // CFL dt of the new cell mean (hodg/timestepping.py:121-134), 3D;
            // threads t < E (element t), no other warp waits
            double dt = 0.0;
            bool okdt = false;
            if (e < ne) {
                double mm[5];
#pragma unroll
                for (int k = 0; k < 5; ++k) {
                    mm[k] = RED[5 * E + k * E + e];
#pragma unroll
                    for (int hh = 1; hh < H; ++hh) mm[k] += RED[5 * E + hh * 5 * E + k * E + e];
                }
                const double m0 = mm[0], m1 = mm[1], m2 = mm[2], m3 = mm[3], m4 = mm[4];
                if (!(m0 > 0.0)) {
                    flag(err, 2, uint32_t(gid));
                } else {
                    const double ri = 1.0 / m0;
                    const double u = m1 * ri, vv = m2 * ri, w = m3 * ri;
                    const double p = (m.gamma - 1.0) * (m4 - 0.5 * m0 * (u * u + vv * vv + w * w));
                    if (!(p > 0.0)) {
                        flag(err, 2, uint32_t(gid));
                    } else {
                        const double speed = sqrt(u * u + vv * vv + w * w) + sqrt(m.gamma * p * ri);
                        dt = a.cfl * G[13 * E + e] / ((2.0 * ORDER + 1.0) * speed);
                        okdt = true;
                    }
                }
                if (a.dt_vec_out) a.dt_vec_out[gid] = dt;
            }
            if (a.dt_next) {
                unsigned long long bits = okdt ? static_cast<unsigned long long>(__double_as_longlong(dt))
                                               : 0x7FF0000000000000ull;
                constexpr int W = E < 32 ? E : 32;
                constexpr unsigned mask = E < 32 ? ((1u << E) - 1u) : 0xffffffffu;  // lanes t < E
#pragma unroll
                for (int o = W / 2; o > 0; o >>= 1) {
                    const unsigned long long other = __shfl_xor_sync(mask, bits, o);
                    bits = other < bits ? other : bits;
                }
                if ((lane % W) == 0) atomicMin(a.dt_next, bits);
            }
        }
        // the output tile is read by the bulk store before the next tile's
        // volume phase overwrites the region
        if (t == 0 && a.combine >= 0 && ne > 0) bulk_wait_read();
        if constexpr (!EPERSIST) break;  // one tile per CTA
    }
}

// ---------------------------------------------------------------------------
// Standalone CFL dt of a state (hodg/timestepping.py:105-147): thread per element.
__global__ void local_dt_kernel(const hodg_mesh_desc m, const double* __restrict__ state, double cfl,
                                double* __restrict__ dt_vec, unsigned long long* __restrict__ dt_min,
                                uint32_t* __restrict__ err) {
    const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool live = c < m.n_elems;
    double dt = 0.0;
    bool ok = false;
    if (live) {
        double mm[5];
#pragma unroll
        for (int v = 0; v < 5; ++v) {
            double s = 0.0;
            sfor<NB>([&](auto j) { s += MEAN_T[j] * state[c * RS + v * NB + j]; });
            mm[v] = s;
        }
        if (!(mm[0] > 0.0)) {
            flag(err, 2, uint32_t(c));
        } else {
            const double u = mm[1] / mm[0], vv = mm[2] / mm[0], w = mm[3] / mm[0];
            const double p = (m.gamma - 1.0) * (mm[4] - 0.5 * mm[0] * (u * u + vv * vv + w * w));
            if (!(p > 0.0)) {
                flag(err, 2, uint32_t(c));
            } else {
                const double speed = sqrt(u * u + vv * vv + w * w) + sqrt(m.gamma * p / mm[0]);
                dt = cfl * m.egeo[(c / E) * 16 * E + 13 * E + (c % E)] / ((2.0 * ORDER + 1.0) * speed);
                ok = true;
            }
        }
        if (dt_vec) dt_vec[c] = dt;
    }
    if (dt_min) {
        // warp min, one atomic per warp (an atomic per element serialises
        // a million same-address updates at the L2)
        unsigned long long bits = ok ? static_cast<unsigned long long>(__double_as_longlong(dt))
                                     : 0x7FF0000000000000ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long other = __shfl_xor_sync(0xffffffffu, bits, o);
            bits = other < bits ? other : bits;
        }
        if ((threadIdx.x & 31) == 0 && bits != 0x7FF0000000000000ull) atomicMin(dt_min, bits);
    }
}

// ---------------------------------------------------------------------------
// Modal transform between the reference's physical Taylor basis b_j(X),
// X = (x - xc)/h (hodg/basis.py), and the reference-element basis m_i(eta):
// b_j(A eta) = sum_i T_ij m_i(eta), A = J/h.  to_reference: c' = T c with A;
// back: c = T(A^-1) c'.  Each column is the product of |alpha_j| linear forms.
__host__ __device__ constexpr int mono_index(int a, int b, int c) {
    const int k = a + b + c;
    return k * (k + 1) * (k + 2) / 6 + (k - a) * (k - a + 1) / 2 + (k - a - b);
}

__global__ void modal_transform_kernel(const hodg_mesh_desc m, int to_reference, const double* __restrict__ in,
                                       double* __restrict__ out) {
    const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= m.n_elems) return;
    double M[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) M[k] = m.econv[c * 18 + (to_reference ? 0 : 9) + k];
    double o[5][NB];
#pragma unroll
    for (int v = 0; v < 5; ++v)
#pragma unroll
        for (int i = 0; i < NB; ++i) o[v][i] = 0.0;
    sfor<NB>([&](auto j) {
        // column j: product of |alpha_j| linear forms sum_m M[d][m] eta_m
        double poly[NB];
#pragma unroll
        for (int i = 0; i < NB; ++i) poly[i] = 0.0;
        poly[0] = 1.0;
        constexpr int f0 = expt(j, 0), f1 = expt(j, 1), f2 = expt(j, 2);
        constexpr int nfac = f0 + f1 + f2;
        sfor<nfac>([&](auto r) {
            constexpr int d = r < f0 ? 0 : (r < f0 + f1 ? 1 : 2);
            constexpr int deg = r;
            double np[NB];
#pragma unroll
            for (int i = 0; i < NB; ++i) np[i] = 0.0;
            sfor<NB>([&](auto i) {
                if constexpr (expt(i, 0) + expt(i, 1) + expt(i, 2) == deg) {
                    sfor<3>([&](auto mm) {
                        constexpr int tgt =
                            mono_index(expt(i, 0) + (mm == 0), expt(i, 1) + (mm == 1), expt(i, 2) + (mm == 2));
                        if constexpr (tgt < NB) np[tgt] += poly[i] * M[d * 3 + mm];
                    });
                }
            });
#pragma unroll
            for (int i = 0; i < NB; ++i) poly[i] = np[i];
        });
#pragma unroll
        for (int v = 0; v < 5; ++v) {
            const double cj = in[c * RS + v * NB + j];
#pragma unroll
            for (int i = 0; i < NB; ++i) o[v][i] += poly[i] * cj;
        }
    });
#pragma unroll
    for (int v = 0; v < 5; ++v)
#pragma unroll
        for (int i = 0; i < NB; ++i) out[c * RS + v * NB + i] = o[v][i];
}

#include "hodg_elem_warp.cuh"

}  // namespace HODG_CAT(ord, ORDER)
}  // namespace hodg

// ---------------------------------------------------------------------------
// host launchers for this order (called by hodg_abi.cu)

namespace hodg {
namespace HODG_CAT(ord, ORDER) {

// per-device launch setup of one kernel: the dynamic shared memory attribute
// and the persistent grid cap (CTAs per SM x SMs) -- a process may drive
// several devices, so both are cached per device
struct LaunchCache {
    int cap[64] = {0};
};
template <typename K>
static int launch_setup(LaunchCache& lc, K kernel, int threads, size_t smem, int* cap) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return HODG_ECUDA;
    if (lc.cap[dev] == 0) {
        const cudaError_t ae = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (ae != cudaSuccess) {
            hodg_note_error(int(ae), 1);
            return HODG_ECUDA;
        }
        int sms = 0, per_sm = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
        lc.cap[dev] = sms * (per_sm > 0 ? per_sm : 1);
    }
    *cap = lc.cap[dev];
    return HODG_OK;
}

// ordinary launch, or a programmatic dependent launch (griddepcontrol) on
// meshes of at most HODG_PDL_MAX_ELEMS elements
template <typename K, typename... Args>
static int launch_maybe_pdl(const hodg_mesh_desc& m, K kernel, int64_t nblk, int threads, size_t smem,
                            cudaStream_t st, Args... args) {
    if (nblk <= 0) return HODG_OK;
    if (HODG_PDL && m.n_elems <= hodg_pdl_max_elems()) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(nblk));
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        const cudaError_t le = cudaLaunchKernelEx(&cfg, kernel, args...);
        if (le != cudaSuccess) {
            hodg_note_error(int(le), 3);
            return HODG_ECUDA;
        }
    } else {
        kernel<<<unsigned(nblk), threads, smem, st>>>(args...);
    }
    const cudaError_t ge = cudaGetLastError();
    if (ge != cudaSuccess) hodg_note_error(int(ge), 4);
    return ge == cudaSuccess ? HODG_OK : HODG_ECUDA;
}

template <typename T, bool BND, bool ES, typename R>
static int launch_face_k(const hodg_mesh_desc& m, const R* state, void* hbuf, uint32_t* err, cudaStream_t st,
                         int64_t fb, int64_t fe) {
    const size_t sm = face_smem_bytes<T, R>();
    static LaunchCache lc;
    int cap = 0;
    if (launch_setup(lc, face_flux_kernel<T, BND, ES, R>, FACE_THREADS, sm, &cap) != HODG_OK) return HODG_ECUDA;
    const int64_t ntiles = (fe - fb + FT - 1) / FT;
    const int64_t nblk = ntiles < cap ? ntiles : cap;  // persistent CTAs loop over tiles
    CUtensorMap rmap = {};
    if (FG4 && nblk > 0 &&
        encode_row_map(&rmap, state, rstride<R>(), int(sizeof(R)),
                       HODG_G4_EXACT ? uint64_t(m.n_elems) : uint64_t(HODG_G4_ROWS)) != HODG_OK)
        return HODG_ECUDA;
    return launch_maybe_pdl(m, face_flux_kernel<T, BND, ES, R>, nblk, FACE_THREADS, sm, st, m, state,
                            static_cast<T*>(hbuf), err, fb, fe, rmap);
}

// interior_only: every face in [fb, fe) has a right element (no boundary
// state code in the kernel)
template <typename T, typename R>
static int launch_face(const hodg_mesh_desc& m, const R* state, void* hbuf, uint32_t* err, cudaStream_t st,
                       int64_t fb, int64_t fe, int interior_only, int es) {
    if (es)
        return interior_only ? launch_face_k<T, false, true, R>(m, state, hbuf, err, st, fb, fe)
                             : launch_face_k<T, true, true, R>(m, state, hbuf, err, st, fb, fe);
    return interior_only ? launch_face_k<T, false, false, R>(m, state, hbuf, err, st, fb, fe)
                         : launch_face_k<T, true, false, R>(m, state, hbuf, err, st, fb, fe);
}

// FP64 state -> its FP32 shadow (rows [0, n_rows), padding zeroed)
__global__ void state_to_f32_kernel(const double* __restrict__ in, int64_t n_rows, float* __restrict__ out) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n_rows * RSF) return;
    const int64_t r = k / RSF;
    const int j = int(k - r * RSF);
    out[k] = j < 5 * NB ? float(in[r * RS + j]) : 0.0f;
}

template <typename T, bool ES>
static int launch_elem_k(const hodg_mesh_desc& m, const void* hbuf, const hodg_stage_args& a, uint32_t* err,
                         cudaStream_t st) {
    if constexpr (WARP_ELEM) {
        // persistent warp groups (hodg_elem_warp.cuh)
        const size_t sm = warp_smem_bytes<T, ES>();
        static LaunchCache lc;
        int cap = 0;
        if (launch_setup(lc, elem_warp_kernel<T, ES>, WPC * 32, sm, &cap) != HODG_OK) return HODG_ECUDA;
        const int64_t need = ((m.n_elems + G - 1) / G + WPC - 1) / WPC;
        const int64_t nblk = need < cap ? need : cap;
        return launch_maybe_pdl(m, elem_warp_kernel<T, ES>, nblk, WPC * 32, sm, st, m, static_cast<const T*>(hbuf),
                                a, err);
    } else {
        const size_t sm = elem_smem_bytes<T, ES>();
        static LaunchCache lc;
        int cap = 0;
        if (launch_setup(lc, elem_stage_kernel<T, ES>, ETHREADS, sm, &cap) != HODG_OK) return HODG_ECUDA;
        const int64_t ntiles = (m.n_elems + E - 1) / E;
        const int64_t nblk = EPERSIST && ntiles > cap ? cap : ntiles;  // persistent CTAs loop over tiles
        CUtensorMap hmap = {};
        if (!ES && elem_g4<T>() && nblk > 0 && encode_row_map(&hmap, hbuf, hstride<T>(), int(sizeof(T))) != HODG_OK)
            return HODG_ECUDA;
        return launch_maybe_pdl(m, elem_stage_kernel<T, ES>, nblk, ETHREADS, sm, st, m, static_cast<const T*>(hbuf),
                                a, err, hmap);
    }
}

template <typename T>
static int launch_elem(const hodg_mesh_desc& m, const void* hbuf, const hodg_stage_args& a, uint32_t* err,
                       cudaStream_t st, int es) {
    return es ? launch_elem_k<T, true>(m, hbuf, a, err, st) : launch_elem_k<T, false>(m, hbuf, a, err, st);
}

}  // namespace HODG_CAT(ord, ORDER)
}  // namespace hodg

extern "C++" {
int HODG_CAT(hodg_launch_face_p, ORDER)(const hodg_mesh_desc& m, int prec, const double* state, void* hbuf,
                                         uint32_t* err, cudaStream_t st, int64_t fb, int64_t fe, int interior,
                                         int es) {
    using namespace hodg::HODG_CAT(ord, ORDER);
    return prec == HODG_PREC_MIXED ? launch_face<float, double>(m, state, hbuf, err, st, fb, fe, interior, es)
                                   : launch_face<double, double>(m, state, hbuf, err, st, fb, fe, interior, es);
}

int HODG_CAT(hodg_launch_face32_p, ORDER)(const hodg_mesh_desc& m, const float* state32, void* hbuf, uint32_t* err,
                                           cudaStream_t st, int64_t fb, int64_t fe, int interior, int es) {
    using namespace hodg::HODG_CAT(ord, ORDER);
    return launch_face<float, float>(m, state32, hbuf, err, st, fb, fe, interior, es);
}

int HODG_CAT(hodg_launch_to_f32_p, ORDER)(const double* rows, int64_t n_rows, float* rows32, cudaStream_t st) {
    using namespace hodg::HODG_CAT(ord, ORDER);
    const int64_t n = n_rows * RSF;
    if (n > 0) state_to_f32_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(rows, n_rows, rows32);
    return cudaGetLastError() == cudaSuccess ? HODG_OK : HODG_ECUDA;
}

int HODG_CAT(hodg_state32_stride_p, ORDER)() { return hodg::HODG_CAT(ord, ORDER)::RSF; }

int HODG_CAT(hodg_launch_elem_p, ORDER)(const hodg_mesh_desc& m, int prec, const void* hbuf,
                                         const hodg_stage_args& a, uint32_t* err, cudaStream_t st, int es) {
    using namespace hodg::HODG_CAT(ord, ORDER);
    return prec == HODG_PREC_MIXED ? launch_elem<float>(m, hbuf, a, err, st, es)
                                   : launch_elem<double>(m, hbuf, a, err, st, es);
}

int HODG_CAT(hodg_elem_record_stride_p, ORDER)() { return hodg::HODG_CAT(ord, ORDER)::EREC; }
int HODG_CAT(hodg_elem_tile_p, ORDER)() { return hodg::HODG_CAT(ord, ORDER)::E; }

int HODG_CAT(hodg_launch_dt_p, ORDER)(const hodg_mesh_desc& m, const double* state, double cfl, double* dt_vec,
                                       unsigned long long* dt_min, uint32_t* err, cudaStream_t st) {
    using namespace hodg::HODG_CAT(ord, ORDER);
    const int64_t nblk = (m.n_elems + 127) / 128;
    if (nblk > 0) local_dt_kernel<<<unsigned(nblk), 128, 0, st>>>(m, state, cfl, dt_vec, dt_min, err);
    return cudaGetLastError() == cudaSuccess ? HODG_OK : HODG_ECUDA;
}

int HODG_CAT(hodg_launch_modal_p, ORDER)(const hodg_mesh_desc& m, int to_ref, const double* in, double* out,
                                          cudaStream_t st) {
    using namespace hodg::HODG_CAT(ord, ORDER);
    const int64_t nblk = (m.n_elems + 127) / 128;
    if (nblk > 0) modal_transform_kernel<<<unsigned(nblk), 128, 0, st>>>(m, to_ref, in, out);
    return cudaGetLastError() == cudaSuccess ? HODG_OK : HODG_ECUDA;
}

int64_t HODG_CAT(hodg_elem_blocks_p, ORDER)(int64_t n) {
    using namespace hodg::HODG_CAT(ord, ORDER);
    return (n + E - 1) / E;
}
}
