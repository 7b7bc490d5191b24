// Shared device code for the tetrahedral DG Euler residual (sm_100a).
//
// Point physics restated from the reference's scalar ops
// (hodg/physics.py:158-344) for 5 conserved variables (rho, rho u, rho v,
// rho w, E): primitive recovery, the Roe flux with the Harten-Hyman entropy
// fix (delta = 0.05 a), the LLF flux, and the far-field / slip / no-slip
// boundary states.  Templated on the arithmetic type so the mixed-precision
// path runs genuine FP32 flux arithmetic.
//
// Also: PTX wrappers for mbarrier + cp.async.bulk (the 1-D TMA engine) used
// to stage element tiles in shared memory.
#pragma once

#include <cuda.h>  // CUtensorMap (encoded through the runtime's driver entry point; no libcuda link)
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include "../../include/hodg_b200.h"

#define HODG_ERR_NONE 0xFFFFFFFFu

// diagnostics: the last failing CUDA / driver code seen by a launcher and
// where (hodg_last_error in hodg_abi.cu); launchers return HODG_ECUDA
extern "C" void hodg_note_error(int code, int site);

namespace hodg {

// ---------------------------------------------------------------------------
// TMA bulk copies and mbarriers (PTX ISA: cp.async.bulk, mbarrier)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

// raise the phase's expected transaction bytes without arriving
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// global -> shared, completion counted on `bar` (bytes % 16 == 0, 16B aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// four rows of a 2-D tensor map (row indices r0..r3; out-of-range rows, e.g.
// -1, are zero-filled without a memory read) -> four consecutive rows at dst
// (128-byte aligned), completion counted on `bar`: one instruction where
// per-row bulk copies take four (sm_100 tile::gather4)
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* tm, int r0, int r1, int r2, int r3,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
        : "memory");
}

// host: the 2-D row map of a row array (rows of `cols` elements, 8- or
// 4-byte, `cols * elem` a multiple of 16 bytes) for tma_gather4: box = one
// full row.  The row count is left open (2^31 - 1): the kernels index only
// valid rows or -1.
#ifndef HODG_G4_ROWS
#define HODG_G4_ROWS 0x7FFFFFFF
#endif
#ifndef HODG_G4_PROMOTION
#define HODG_G4_PROMOTION CU_TENSOR_MAP_L2_PROMOTION_NONE
#endif
static inline int encode_row_map(CUtensorMap* tm, const void* base, int cols, int elem_bytes,
                                 uint64_t rows = HODG_G4_ROWS) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !enc)
            return HODG_ECUDA;
    }
    const cuuint64_t gdim[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    const cuuint64_t gstride[1] = {cuuint64_t(cols) * elem_bytes};
    const cuuint32_t box[2] = {cuuint32_t(cols), 1};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = enc(tm, elem_bytes == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                           const_cast<void*>(base), gdim, gstride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, HODG_G4_PROMOTION,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) hodg_note_error(int(r), 2);
    return r == CUDA_SUCCESS ? HODG_OK : HODG_ECUDA;
}

// global -> L2 prefetch of a contiguous range (no completion tracking)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// shared -> global (bulk group); caller waits with bulk_wait_read()
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}


// 16-byte global -> shared copy by the calling thread (cp.async, L2 only);
// completion per thread with cp_async_wait_all(), then a barrier among the
// threads that read the destination
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// one arrival on `bar` once all of this thread's prior cp.async copies landed
// (counts against the barrier's expected arrivals: .noinc)
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// make generic-proxy smem writes visible to the async (TMA) proxy
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------------------
// error words: err[0] first inadmissible face, err[1] first inadmissible
// volume point's cell, err[2] first inadmissible cell mean (dt pass)

__device__ __forceinline__ void flag(uint32_t* err, int which, uint32_t id) {
    if (err) atomicMin(err + which, id);
}

// ---------------------------------------------------------------------------
// point physics

template <typename T>
struct K {
    static constexpr T one = T(1), half = T(0.5), two = T(2), quarter = T(0.25), efix = T(0.05), zero = T(0);
};

#ifndef HODG_F32_FAST_RCP
#define HODG_F32_FAST_RCP 1
#endif
// Reciprocal and reciprocal square root on the hot paths: in FP64 the MUFU
// approximation (rcp / rsqrt.approx.ftz.f64, ~2^-22 relative) refined by two
// Newton steps (quadratic: ~2^-86, i.e. a 1-ulp result) -- no special-case
// branches and no correctly-rounded division sequence.  Arguments are
// positive normal numbers on admissible states; an inadmissible state
// (rho, p or a^2 <= 0) yields garbage that the callers' ok flags discard.
// FP32 keeps the IEEE operations.
__device__ __forceinline__ double rcp_nr(double d) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    double e = fma(-d, y, 1.0);
    y = fma(y, e, y);
    e = fma(-d, y, 1.0);
    return fma(y, e, y);
}
__device__ __forceinline__ double rsqrt_nr(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double r = fma(-x * y, y, 1.0);
    y = fma(0.5 * y, r, y);
    r = fma(-x * y, y, 1.0);
    return fma(0.5 * y, r, y);
}
__device__ __forceinline__ float rcp_nr(float d) {
#if HODG_F32_FAST_RCP
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(d));
    return fmaf(y, fmaf(-d, y, 1.0f), y);  // one Newton step: ~1 ulp
#else
    return 1.0f / d;
#endif
}
__device__ __forceinline__ float rsqrt_nr(float x) { return rsqrtf(x); }

// primitive (u, v, w, p) from conserved; hodg/physics.py:159-165
template <typename T>
__device__ __forceinline__ T prim(const T q[5], T g, T& u, T& v, T& w) {
    T ri = rcp_nr(q[0]);
    u = q[1] * ri;
    v = q[2] * ri;
    w = q[3] * ri;
    return (g - K<T>::one) * (q[4] - K<T>::half * q[0] * (u * u + v * v + w * w));
}

// Roe flux with Harten-Hyman entropy fix; hodg/physics.py:177-250 (3D).
// Straight-line (no early returns, entropy fix as selects) so two calls
// interleave; divisions and square roots are replaced by rsqrt(rho) per
// side (sqrt(rho) = rho rsqrt, 1/rho = rsqrt^2), 1/(sL + sR) and rsqrt(a2).  Returns ok = 0 on rho <= 0, p <= 0 or a2 <= 0 (then f is
// garbage and the caller flags the face, as the reference's ok = 0).
template <typename T>
__device__ __forceinline__ bool roe(const T qL[5], const T qR[5], const T n[3], T g, T f[5]) {
    const T one = K<T>::one, half = K<T>::half;
    // one rsqrt per side gives both sqrt(rho) and 1/rho
    const T isL = rsqrt_nr(qL[0]), isR = rsqrt_nr(qR[0]);
    const T riL = isL * isL, riR = isR * isR;
    const T sL = qL[0] * isL, sR = qR[0] * isR;
    const T uL = qL[1] * riL, vL = qL[2] * riL, wL = qL[3] * riL;
    const T uR = qR[1] * riR, vR = qR[2] * riR, wR = qR[3] * riR;
    const T gm1 = g - one;
    const T pL = gm1 * (qL[4] - half * qL[0] * (uL * uL + vL * vL + wL * wL));
    const T pR = gm1 * (qR[4] - half * qR[0] * (uR * uR + vR * vR + wR * wR));
    const T nx = n[0], ny = n[1], nz = n[2];
    const T vnL = uL * nx + vL * ny + wL * nz;
    const T vnR = uR * nx + vR * ny + wR * nz;
    const T di = rcp_nr(sL + sR);
    const T ut = (sL * uL + sR * uR) * di;
    const T vt = (sL * vL + sR * vR) * di;
    const T wt = (sL * wL + sR * wR) * di;
    const T HL = (qL[4] + pL) * riL;
    const T HR = (qR[4] + pR) * riR;
    const T Ht = (sL * HL + sR * HR) * di;
    const T ke = half * (ut * ut + vt * vt + wt * wt);
    const T a2 = gm1 * (Ht - ke);
    const bool ok = (qL[0] > T(0)) & (qR[0] > T(0)) & (pL > T(0)) & (pR > T(0)) & (a2 > T(0));
    const T ra = rsqrt_nr(a2);
    const T a = a2 * ra;
    const T rt = sL * sR;
    const T unt = ut * nx + vt * ny + wt * nz;
    const T dr = qR[0] - qL[0];
    const T dp = pR - pL;
    const T du = uR - uL, dv = vR - vL, dw = wR - wL;
    const T dun = vnR - vnL;
    T l1 = fabs(unt - a), l4 = fabs(unt + a);
    const T l2 = fabs(unt);
    const T delta = K<T>::efix * a;
    const T idelta = (one / K<T>::efix) * ra;
    l1 = (l1 < delta) ? half * (l1 * l1 * idelta + delta) : l1;
    l4 = (l4 < delta) ? half * (l4 * l4 * idelta + delta) : l4;
    const T ia2h = half * ra * ra;
    const T rad = rt * a * dun;
    const T a1 = (dp - rad) * ia2h;
    const T a4 = (dp + rad) * ia2h;
    const T a2w = dr - dp * (ra * ra);
    const T w1 = l1 * a1, w4 = l4 * a4;
    // dissipation sum_k |lambda_k| alpha_k r_k, with the acoustic pair
    // (w1, w4) and the shear/entropy terms regrouped by ut / n / du:
    //   d_x = d0 ut + cn nx + l2 rt du,  cn = (w4 - w1) a - l2 rt dun,
    //   dE  = (w1 + w4) Ht + l2 a2w ke + cn unt + l2 rt (ut du + vt dv + wt dw)
    const T sw = w1 + w4;
    const T l2a2w = l2 * a2w;
    const T l2rt = l2 * rt;
    const T d0 = sw + l2a2w;
    const T cn = (w4 - w1) * a - l2rt * dun;
    const T d1 = d0 * ut + cn * nx + l2rt * du;
    const T d2 = d0 * vt + cn * ny + l2rt * dv;
    const T d3 = d0 * wt + cn * nz + l2rt * dw;
    const T dE = sw * Ht + l2a2w * ke + cn * unt + l2rt * (ut * du + vt * dv + wt * dw);
    f[0] = half * (qL[0] * vnL + qR[0] * vnR - d0);
    f[1] = half * (qL[1] * vnL + qR[1] * vnR + (pL + pR) * nx - d1);
    f[2] = half * (qL[2] * vnL + qR[2] * vnR + (pL + pR) * ny - d2);
    f[3] = half * (qL[3] * vnL + qR[3] * vnR + (pL + pR) * nz - d3);
    f[4] = half * ((qL[4] + pL) * vnL + (qR[4] + pR) * vnR - dE);
    return ok;
}

// FP32 Roe-HH with the left / right states in packed f32x2 lanes (sm_100
// FFMA2 / FMUL2 / FADD2: two operations per issue slot).  Same formulas as
// roe<float>; the one-sided quantities (sqrt rho, 1/rho, velocities, p, H,
// normal velocity) and the paired terms of the dissipation and the flux are
// evaluated two at a time.
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 f2b(float a) { return make_float2(a, a); }
__device__ __forceinline__ bool roe_x2(const float qL[5], const float qR[5], const float n[3], float g, float f[5]) {
    const float2 q0 = f2(qL[0], qR[0]), q1 = f2(qL[1], qR[1]), q2 = f2(qL[2], qR[2]), q3 = f2(qL[3], qR[3]),
                 q4 = f2(qL[4], qR[4]);
    const float2 is = f2(rsqrtf(qL[0]), rsqrtf(qR[0]));
    const float2 ri = __fmul2_rn(is, is);
    const float2 sq = __fmul2_rn(q0, is);  // sqrt(rho)
    const float2 u = __fmul2_rn(q1, ri), v = __fmul2_rn(q2, ri), w = __fmul2_rn(q3, ri);
    const float gm1 = g - 1.0f;
    const float2 k2 = __ffma2_rn(w, w, __ffma2_rn(v, v, __fmul2_rn(u, u)));      // |u|^2
    const float2 p = __fmul2_rn(f2b(gm1), __ffma2_rn(__fmul2_rn(f2b(-0.5f), q0), k2, q4));
    const float nx = n[0], ny = n[1], nz = n[2];
    const float2 vn = __ffma2_rn(w, f2b(nz), __ffma2_rn(v, f2b(ny), __fmul2_rn(u, f2b(nx))));
    const float2 hh = __fmul2_rn(__fadd2_rn(q4, p), ri);                         // total enthalpy
    const float di = rcp_nr(sq.x + sq.y);
    // Roe averages: (sL xL + sR xR) / (sL + sR), two quantities per pair
    const float2 su = __fmul2_rn(sq, u), sv = __fmul2_rn(sq, v), sw_ = __fmul2_rn(sq, w), sh = __fmul2_rn(sq, hh);
    const float2 uv = __fmul2_rn(f2(su.x + su.y, sv.x + sv.y), f2b(di));
    const float2 wh = __fmul2_rn(f2(sw_.x + sw_.y, sh.x + sh.y), f2b(di));
    const float ut = uv.x, vt = uv.y, wt = wh.x, Ht = wh.y;
    const float ke = 0.5f * (ut * ut + vt * vt + wt * wt);
    const float a2 = gm1 * (Ht - ke);
    const bool ok = (qL[0] > 0.0f) & (qR[0] > 0.0f) & (p.x > 0.0f) & (p.y > 0.0f) & (a2 > 0.0f);
    const float ra = rsqrtf(a2);
    const float a = a2 * ra;
    const float rt = sq.x * sq.y;
    const float unt = ut * nx + vt * ny + wt * nz;
    const float dr = qR[0] - qL[0];
    const float dp = p.y - p.x;
    const float du = u.y - u.x, dv = v.y - v.x, dw = w.y - w.x;
    const float dun = vn.y - vn.x;
    // acoustic pair (l1, l4) with the Harten-Hyman fix
    float2 l14 = __fadd2_rn(f2b(unt), f2(-a, a));
    l14.x = fabsf(l14.x);
    l14.y = fabsf(l14.y);
    const float l2 = fabsf(unt);
    const float delta = 0.05f * a;
    const float idelta = (1.0f / 0.05f) * ra;
    const float2 fix = __fmul2_rn(f2b(0.5f), __ffma2_rn(__fmul2_rn(l14, l14), f2b(idelta), f2b(delta)));
    l14.x = l14.x < delta ? fix.x : l14.x;
    l14.y = l14.y < delta ? fix.y : l14.y;
    const float ia2h = 0.5f * ra * ra;
    const float rad = rt * a * dun;
    const float2 a14 = __fmul2_rn(__fadd2_rn(f2b(dp), f2(-rad, rad)), f2b(ia2h));
    const float a2w = dr - dp * (ra * ra);
    const float2 w14 = __fmul2_rn(l14, a14);
    const float sw = w14.x + w14.y;
    const float l2a2w = l2 * a2w;
    const float l2rt = l2 * rt;
    const float d0 = sw + l2a2w;
    const float cn = (w14.y - w14.x) * a - l2rt * dun;
    const float2 d12 = __ffma2_rn(f2b(l2rt), f2(du, dv), __ffma2_rn(f2b(cn), f2(nx, ny), __fmul2_rn(f2b(d0), uv)));
    const float d3 = d0 * wt + cn * nz + l2rt * dw;
    const float dE = sw * Ht + l2a2w * ke + cn * unt + l2rt * (ut * du + vt * dv + wt * dw);
    const float ps = p.x + p.y;
    // central part: qL vnL + qR vnR (+ p n) per variable, two variables per pair
    const float2 c01 = __ffma2_rn(f2(qR[0], qR[1]), f2b(vn.y), __fmul2_rn(f2(qL[0], qL[1]), f2b(vn.x)));
    const float2 c23 = __ffma2_rn(f2(qR[2], qR[3]), f2b(vn.y), __fmul2_rn(f2(qL[2], qL[3]), f2b(vn.x)));
    const float c4 = (qL[4] + p.x) * vn.x + (qR[4] + p.y) * vn.y;
    const float2 f01 = __fmul2_rn(f2b(0.5f), __fadd2_rn(__fadd2_rn(c01, f2(0.0f, ps * nx)), f2(-d0, -d12.x)));
    const float2 f23 = __fmul2_rn(f2b(0.5f), __fadd2_rn(__ffma2_rn(f2b(ps), f2(ny, nz), c23), f2(-d12.y, -d3)));
    f[0] = f01.x;
    f[1] = f01.y;
    f[2] = f23.x;
    f[3] = f23.y;
    f[4] = 0.5f * (c4 - dE);
    return ok;
}

// local Lax-Friedrichs (Rusanov) flux
template <typename T>
__device__ __forceinline__ bool llf(const T qL[5], const T qR[5], const T n[3], T g, T f[5]) {
    if (!(qL[0] > K<T>::zero) || !(qR[0] > K<T>::zero)) return false;
    T uL, vL, wL, uR, vR, wR;
    T pL = prim(qL, g, uL, vL, wL);
    T pR = prim(qR, g, uR, vR, wR);
    if (!(pL > K<T>::zero) || !(pR > K<T>::zero)) return false;
    T vnL = uL * n[0] + vL * n[1] + wL * n[2];
    T vnR = uR * n[0] + vR * n[1] + wR * n[2];
    T sl = fabs(vnL) + sqrt(g * pL / qL[0]);
    T sr = fabs(vnR) + sqrt(g * pR / qR[0]);
    T lam = sl > sr ? sl : sr;
    T FL[5] = {qL[0] * vnL, qL[1] * vnL + pL * n[0], qL[2] * vnL + pL * n[1], qL[3] * vnL + pL * n[2],
               (qL[4] + pL) * vnL};
    T FR[5] = {qR[0] * vnR, qR[1] * vnR + pR * n[0], qR[2] * vnR + pR * n[1], qR[3] * vnR + pR * n[2],
               (qR[4] + pR) * vnR};
#pragma unroll
    for (int v = 0; v < 5; ++v) f[v] = K<T>::half * (FL[v] + FR[v]) - K<T>::half * lam * (qR[v] - qL[v]);
    return true;
}

// boundary states; hodg/physics.py:292-344 with a 3-vector tangential velocity
template <typename T>
__device__ __forceinline__ void bstate(int kind, const T q[5], const T n[3], const T qf[5], T g, T out[5]) {
    const T one = K<T>::one, two = K<T>::two, half = K<T>::half;
    if (kind == HODG_BC_FAR_FIELD) {
        T ui, vi, wi, uf, vf, wf;
        T pi = prim(q, g, ui, vi, wi);
        T pf = prim(qf, g, uf, vf, wf);
        T ai = sqrt(g * pi / q[0]);
        T af = sqrt(g * pf / qf[0]);
        T uni = ui * n[0] + vi * n[1] + wi * n[2];
        T unf = uf * n[0] + vf * n[1] + wf * n[2];
        if (uni >= ai) {
#pragma unroll
            for (int v = 0; v < 5; ++v) out[v] = q[v];
            return;
        }
        if (unf <= -af) {
#pragma unroll
            for (int v = 0; v < 5; ++v) out[v] = qf[v];
            return;
        }
        T gm1i = one / (g - one);
        T rplus = uni + two * ai * gm1i;
        T rminus = unf - two * af * gm1i;
        T unb = half * (rplus + rminus);
        T ab = K<T>::quarter * (g - one) * (rplus - rminus);
        if (!(ab > K<T>::zero)) {
#pragma unroll
            for (int v = 0; v < 5; ++v) out[v] = qf[v];
            return;
        }
        T s, utx, uty, utz;
        if (unb > K<T>::zero) {
            s = pi / pow(q[0], g);
            utx = ui - uni * n[0];
            uty = vi - uni * n[1];
            utz = wi - uni * n[2];
        } else {
            s = pf / pow(qf[0], g);
            utx = uf - unf * n[0];
            uty = vf - unf * n[1];
            utz = wf - unf * n[2];
        }
        T rb = pow(ab * ab / (g * s), gm1i);
        T pb = rb * ab * ab / g;
        T ub = utx + unb * n[0], vb = uty + unb * n[1], wb = utz + unb * n[2];
        out[0] = rb;
        out[1] = rb * ub;
        out[2] = rb * vb;
        out[3] = rb * wb;
        out[4] = pb * gm1i + half * rb * (ub * ub + vb * vb + wb * wb);
    } else if (kind == HODG_BC_SLIP_WALL) {
        T un2 = two * (q[1] * n[0] + q[2] * n[1] + q[3] * n[2]);
        out[0] = q[0];
        out[1] = q[1] - un2 * n[0];
        out[2] = q[2] - un2 * n[1];
        out[3] = q[3] - un2 * n[2];
        out[4] = q[4];
    } else {  // no-slip (also any unknown code, as the reference)
        out[0] = q[0];
        out[1] = -q[1];
        out[2] = -q[2];
        out[3] = -q[3];
        out[4] = q[4];
    }
}

}  // namespace hodg
