// 2D table-driven kernels: the reference's own discretisation (quads and
// triangles, 4 variables, per-cell quadrature tables from
// hodg/geometry.py:120-220) on the GPU, with the reference kernels'
// argument lists -- a literal drop-in for _KERNELS[dtype].flux_pass /
// rhs_pass (hodg/dg.py:240-460), _dt_pass, _axpy_state and _combine_state
// (hodg/timestepping.py:105-180).
//
// Built with -fmad=false and IEEE division / sqrt: the expression trees
// follow the reference's numba code (which emits no FMA), so results match
// the reference bit for bit except where CUDA's pow differs from glibc's by
// an ulp (far-field boundary state).  This is the GPU path that reproduces
// the reference's golden residual histories (tests/test_gpu_2d.py).
// Thread per face / per cell, as the reference's prange loops.
#include <cstdint>

#include "../../include/hodg_b200.h"
#include <cuda_runtime.h>

extern int64_t hodg_count_launch(int64_t n);

namespace {

template <typename T>
struct C2 {
    static constexpr T one = T(1), zero = T(0), half = T(0.5), two = T(2), quarter = T(0.25), efix = T(0.05);
};

// hodg/physics.py:159-165
template <typename T>
__device__ __forceinline__ T prim2(T rho, T ru, T rv, T e, T g, T& u, T& v) {
    u = ru / rho;
    v = rv / rho;
    return (g - C2<T>::one) * (e - C2<T>::half * rho * (u * u + v * v));
}

// hodg/physics.py:177-250
template <typename T>
__device__ bool roe2(const T* qL, const T* qR, T nx, T ny, T g, T* f) {
    const T one = C2<T>::one, half = C2<T>::half, two = C2<T>::two, zero = C2<T>::zero;
    const T rL = qL[0], ruL = qL[1], rvL = qL[2], eL = qL[3];
    const T rR = qR[0], ruR = qR[1], rvR = qR[2], eR = qR[3];
    if (rL <= zero || rR <= zero) return false;
    T uL, vL, uR, vR;
    const T pL = prim2(rL, ruL, rvL, eL, g, uL, vL);
    const T pR = prim2(rR, ruR, rvR, eR, g, uR, vR);
    if (pL <= zero || pR <= zero) return false;
    const T vnL = uL * nx + vL * ny, vnR = uR * nx + vR * ny;
    const T fL0 = rL * vnL, fL1 = ruL * vnL + pL * nx, fL2 = rvL * vnL + pL * ny, fL3 = (eL + pL) * vnL;
    const T fR0 = rR * vnR, fR1 = ruR * vnR + pR * nx, fR2 = rvR * vnR + pR * ny, fR3 = (eR + pR) * vnR;
    const T sL = sqrt(rL);
    const T sR = sqrt(rR);
    const T den = sL + sR;
    const T ut = (sL * uL + sR * uR) / den;
    const T vt = (sL * vL + sR * vR) / den;
    const T HL = (eL + pL) / rL;
    const T HR = (eR + pR) / rR;
    const T Ht = (sL * HL + sR * HR) / den;
    const T ke = half * (ut * ut + vt * vt);
    const T a2 = (g - one) * (Ht - ke);
    if (a2 <= zero) return false;
    const T a = sqrt(a2);
    const T rt = sL * sR;
    const T unt = ut * nx + vt * ny;
    const T dr = rR - rL, dp = pR - pL, du = uR - uL, dv = vR - vL;
    const T dun = (uR * nx + vR * ny) - (uL * nx + vL * ny);
    T l1 = fabs(unt - a);
    const T l2 = fabs(unt);
    T l4 = fabs(unt + a);
    const T delta = C2<T>::efix * a;
    if (l1 < delta) l1 = half * (l1 * l1 / delta + delta);
    if (l4 < delta) l4 = half * (l4 * l4 / delta + delta);
    const T a1 = (dp - rt * a * dun) / (two * a2);
    const T a4 = (dp + rt * a * dun) / (two * a2);
    const T a2w = dr - dp / a2;
    const T d0 = l1 * a1 + l2 * a2w + l4 * a4;
    const T d1 = l1 * a1 * (ut - a * nx) + l2 * (a2w * ut + rt * (du - dun * nx)) + l4 * a4 * (ut + a * nx);
    const T d2 = l1 * a1 * (vt - a * ny) + l2 * (a2w * vt + rt * (dv - dun * ny)) + l4 * a4 * (vt + a * ny);
    const T d3 = l1 * a1 * (Ht - a * unt) + l2 * (a2w * ke + rt * (ut * du + vt * dv - unt * dun)) +
                 l4 * a4 * (Ht + a * unt);
    f[0] = half * (fL0 + fR0) - half * d0;
    f[1] = half * (fL1 + fR1) - half * d1;
    f[2] = half * (fL2 + fR2) - half * d2;
    f[3] = half * (fL3 + fR3) - half * d3;
    return true;
}

// LLF (not in the reference; same definition as the 3D kernels)
template <typename T>
__device__ bool llf2(const T* qL, const T* qR, T nx, T ny, T g, T* f) {
    const T zero = C2<T>::zero, half = C2<T>::half;
    if (qL[0] <= zero || qR[0] <= zero) return false;
    T uL, vL, uR, vR;
    const T pL = prim2(qL[0], qL[1], qL[2], qL[3], g, uL, vL);
    const T pR = prim2(qR[0], qR[1], qR[2], qR[3], g, uR, vR);
    if (pL <= zero || pR <= zero) return false;
    const T vnL = uL * nx + vL * ny, vnR = uR * nx + vR * ny;
    const T sl = fabs(vnL) + sqrt(g * pL / qL[0]), sr = fabs(vnR) + sqrt(g * pR / qR[0]);
    const T lam = sl > sr ? sl : sr;
    const T FL[4] = {qL[0] * vnL, qL[1] * vnL + pL * nx, qL[2] * vnL + pL * ny, (qL[3] + pL) * vnL};
    const T FR[4] = {qR[0] * vnR, qR[1] * vnR + pR * nx, qR[2] * vnR + pR * ny, (qR[3] + pR) * vnR};
    for (int v = 0; v < 4; ++v) f[v] = half * (FL[v] + FR[v]) - half * lam * (qR[v] - qL[v]);
    return true;
}

// x ** y as the reference evaluates it (glibc pow / powf): in FP32 through
// double precision, which rounds to glibc's (correctly rounded) powf except
// in astronomically rare near-tie cases; CUDA's own powf is off by an ulp
// often enough to desynchronise the FP32 fixture histories
__device__ __forceinline__ double ref_pow(double x, double y) { return pow(x, y); }
__device__ __forceinline__ float ref_pow(float x, float y) { return float(pow(double(x), double(y))); }

// hodg/physics.py:292-344
template <typename T>
__device__ void bstate2(int kind, const T* q, T nx, T ny, const T* qf, T g, T* out) {
    const T one = C2<T>::one, two = C2<T>::two, half = C2<T>::half, zero = C2<T>::zero;
    if (kind == HODG_BC_FAR_FIELD) {
        const T rho = q[0], ru = q[1], rv = q[2], e = q[3];
        const T rf = qf[0], ruf = qf[1], rvf = qf[2], ef = qf[3];
        T ui, vi, uf, vf;
        const T pi = prim2(rho, ru, rv, e, g, ui, vi);
        const T pf = prim2(rf, ruf, rvf, ef, g, uf, vf);
        const T ai = sqrt(g * pi / rho);
        const T af = sqrt(g * pf / rf);
        const T uni = ui * nx + vi * ny;
        const T unf = uf * nx + vf * ny;
        if (uni >= ai) {
            for (int v = 0; v < 4; ++v) out[v] = q[v];
            return;
        }
        if (unf <= -af) {
            for (int v = 0; v < 4; ++v) out[v] = qf[v];
            return;
        }
        const T rplus = uni + two * ai / (g - one);
        const T rminus = unf - two * af / (g - one);
        const T unb = half * (rplus + rminus);
        const T ab = C2<T>::quarter * (g - one) * (rplus - rminus);
        if (!(ab > zero)) {
            for (int v = 0; v < 4; ++v) out[v] = qf[v];
            return;
        }
        T s, utx, uty;
        if (unb > zero) {
            s = pi / ref_pow(rho, g);
            utx = ui - uni * nx;
            uty = vi - uni * ny;
        } else {
            s = pf / ref_pow(rf, g);
            utx = uf - unf * nx;
            uty = vf - unf * ny;
        }
        const T rb = ref_pow(ab * ab / (g * s), one / (g - one));
        const T pb = rb * ab * ab / g;
        const T ub = utx + unb * nx;
        const T vb = uty + unb * ny;
        out[0] = rb;
        out[1] = rb * ub;
        out[2] = rb * vb;
        out[3] = pb / (g - one) + half * rb * (ub * ub + vb * vb);
    } else if (kind == HODG_BC_SLIP_WALL) {
        const T un2 = two * (q[1] * nx + q[2] * ny);
        out[0] = q[0];
        out[1] = q[1] - un2 * nx;
        out[2] = q[2] - un2 * ny;
        out[3] = q[3];
    } else {
        out[0] = q[0];
        out[1] = -q[1];
        out[2] = -q[2];
        out[3] = q[3];
    }
}

// hodg/physics.py:252-269 -> (u, v, ux, uy, vx, vy, Tx, Ty)
template <typename T>
__device__ __forceinline__ void vel_temp_grads2(T rho, T ru, T rv, T e, const T* zx, const T* zy, T g, T R, T* o) {
    const T u = ru / rho;
    const T v = rv / rho;
    const T ux = (zx[1] - u * zx[0]) / rho;
    const T vx = (zx[2] - v * zx[0]) / rho;
    const T uy = (zy[1] - u * zy[0]) / rho;
    const T vy = (zy[2] - v * zy[0]) / rho;
    const T ke = C2<T>::half * (u * u + v * v);
    const T ein = e - rho * ke;
    const T kx = ke * zx[0] + rho * (u * ux + v * vx);
    const T ky = ke * zy[0] + rho * (u * uy + v * vy);
    const T coef = (g - C2<T>::one) / R;
    o[0] = u;
    o[1] = v;
    o[2] = ux;
    o[3] = uy;
    o[4] = vx;
    o[5] = vy;
    o[6] = coef * ((zx[3] - kx) * rho - ein * zx[0]) / (rho * rho);
    o[7] = coef * ((zy[3] - ky) * rho - ein * zy[0]) / (rho * rho);
}

// hodg/physics.py:271-277 -> (txx, txy, tyy, qx, qy)
template <typename T>
__device__ __forceinline__ void stress_heat2(const T* gr, T g, T R, T mu, T Pr, T* s) {
    const T two_thirds = T(2.0 / 3.0);
    const T ux = gr[2], uy = gr[3], vx = gr[4], vy = gr[5];
    s[0] = mu * two_thirds * (C2<T>::two * ux - vy);
    s[2] = mu * two_thirds * (C2<T>::two * vy - ux);
    s[1] = mu * (uy + vx);
    const T k = mu * g * R / ((g - C2<T>::one) * Pr);
    s[3] = -k * gr[6];
    s[4] = -k * gr[7];
}

// hodg/physics.py:279-290
template <typename T>
__device__ __forceinline__ void viscn2(const T* q, const T* zx, const T* zy, T nx, T ny, T g, T R, T mu, T Pr,
                                       T* h) {
    T gr[8], s[5];
    vel_temp_grads2(q[0], q[1], q[2], q[3], zx, zy, g, R, gr);
    stress_heat2(gr, g, R, mu, Pr, s);
    const T u = gr[0], v = gr[1];
    h[0] = C2<T>::zero;
    h[1] = s[0] * nx + s[1] * ny;
    h[2] = s[1] * nx + s[2] * ny;
    h[3] = (u * s[0] + v * s[1] - s[3]) * nx + (u * s[1] + v * s[2] - s[4]) * ny;
}

// trace of the 4 variables of `src` (cell-major (.., 4, nb)) at one point
template <typename T>
__device__ __forceinline__ void trace4(const T* __restrict__ b, const T* __restrict__ src, int nb, T* out) {
    for (int v = 0; v < 4; ++v) out[v] = C2<T>::zero;
    for (int k = 0; k < nb; ++k) {
        const T bk = b[k];
        for (int v = 0; v < 4; ++v) out[v] += bk * src[v * nb + k];
    }
}

// hodg/dg.py:114-162 (qhat_pass): thread per face
template <typename T>
__global__ void qhat_pass2d(int64_t n_faces, int nqf, int nb, const T* __restrict__ coeffs, const T* __restrict__ fbL,
                            const T* __restrict__ fbR, const int32_t* __restrict__ face_cells,
                            const int8_t* __restrict__ bc_code, const T* __restrict__ fnx, const T* __restrict__ fny,
                            const T* __restrict__ qinf, double gamma, T* __restrict__ qhat,
                            uint8_t* __restrict__ errf) {
    const int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (f >= n_faces) return;
    const T g = T(gamma);
    const int64_t iL = face_cells[2 * f], iR = face_cells[2 * f + 1];
    const T nx = fnx[f], ny = fny[f];
    for (int q = 0; q < nqf; ++q) {
        T qL[4], qR[4];
        trace4(fbL + (f * nqf + q) * nb, coeffs + iL * 4 * nb, nb, qL);
        if (iR >= 0) {
            trace4(fbR + (f * nqf + q) * nb, coeffs + iR * 4 * nb, nb, qR);
        } else {
            if (qL[0] <= C2<T>::zero) {
                errf[f] = 1;
                continue;
            }
            T u, v;
            if (prim2(qL[0], qL[1], qL[2], qL[3], g, u, v) <= C2<T>::zero) {
                errf[f] = 1;
                continue;
            }
            const T qf[4] = {qinf[0], qinf[1], qinf[2], qinf[3]};
            bstate2(bc_code[f], qL, nx, ny, qf, g, qR);
        }
        for (int v = 0; v < 4; ++v) qhat[(f * nqf + q) * 4 + v] = C2<T>::half * (qL[v] + qR[v]);
    }
}

// hodg/dg.py:164-238 (aux_pass): BR1 weak gradient, thread per cell,
// accumulated and solved at T as the reference's scratch / minv
template <typename T>
__global__ void aux_pass2d(int64_t n_cells, int nb, int nqv, int nqf, int maxf, const T* __restrict__ coeffs,
                           const T* __restrict__ qhat, const T* __restrict__ vol_w, const T* __restrict__ vol_basis,
                           const T* __restrict__ vol_gx, const T* __restrict__ vol_gy,
                           const int8_t* __restrict__ cell_nfaces, const int32_t* __restrict__ cell_faces,
                           const int8_t* __restrict__ cell_fsign, const T* __restrict__ face_w,
                           const T* __restrict__ fbL, const T* __restrict__ fbR, const T* __restrict__ fnx,
                           const T* __restrict__ fny, const T* __restrict__ minv, T* __restrict__ aux) {
    const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= n_cells) return;
    T sc[2 * 4 * 6];
    for (int i = 0; i < 8 * nb; ++i) sc[i] = C2<T>::zero;
    const T* cc = coeffs + c * 4 * nb;
    for (int qp = 0; qp < nqv; ++qp) {
        const T w = vol_w[c * nqv + qp];
        if (w == C2<T>::zero) continue;
        T qv[4];
        trace4(vol_basis + (c * nqv + qp) * nb, cc, nb, qv);
        for (int j = 0; j < nb; ++j) {
            const T gx = w * vol_gx[(c * nqv + qp) * nb + j];
            const T gy = w * vol_gy[(c * nqv + qp) * nb + j];
            for (int v = 0; v < 4; ++v) sc[v * nb + j] -= qv[v] * gx;
            for (int v = 0; v < 4; ++v) sc[(4 + v) * nb + j] -= qv[v] * gy;
        }
    }
    for (int slot = 0; slot < cell_nfaces[c]; ++slot) {
        const int64_t fid = cell_faces[c * maxf + slot];
        const int sgn = cell_fsign[c * maxf + slot];
        const T* tb = sgn > 0 ? fbL : fbR;
        const T s = T(sgn);
        const T nx = fnx[fid], ny = fny[fid];
        for (int q = 0; q < nqf; ++q) {
            const T w = s * face_w[fid * nqf + q];
            const T* h = qhat + (fid * nqf + q) * 4;
            const T wx = w * nx;
            const T wy = w * ny;
            for (int j = 0; j < nb; ++j) {
                const T b = tb[(fid * nqf + q) * nb + j];
                for (int v = 0; v < 4; ++v) sc[v * nb + j] += h[v] * wx * b;
                for (int v = 0; v < 4; ++v) sc[(4 + v) * nb + j] += h[v] * wy * b;
            }
        }
    }
    const T* mi = minv + c * nb * nb;
    for (int dv = 0; dv < 8; ++dv)
        for (int j = 0; j < nb; ++j) {
            T acc = C2<T>::zero;
            for (int k = 0; k < nb; ++k) acc += mi[j * nb + k] * sc[dv * nb + k];
            aux[(c * 8 + dv) * nb + j] = acc;
        }
}

// hodg/dg.py:240-351: thread per face; VIS = the ivis == 1 branch
template <typename T, bool VIS>
__global__ void flux_pass2d(int64_t n_faces, int nqf, int nb, const T* __restrict__ coeffs, const T* __restrict__ aux,
                            const T* __restrict__ fbL, const T* __restrict__ fbR,
                            const int32_t* __restrict__ face_cells, const int8_t* __restrict__ bc_code,
                            const T* __restrict__ fnx, const T* __restrict__ fny, const T* __restrict__ qinf,
                            double gamma, double Rgas, double mu, double Pr, int flux_kind, T* __restrict__ finv,
                            T* __restrict__ fvis, T* __restrict__ fqhat, uint8_t* __restrict__ errf) {
    const int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (f >= n_faces) return;
    const T g = T(gamma);
    const T R = T(Rgas), m = T(mu), pr = T(Pr);
    const int64_t iL = face_cells[2 * f], iR = face_cells[2 * f + 1];
    const T nx = fnx[f], ny = fny[f];
    for (int q = 0; q < nqf; ++q) {
        T qL[4] = {C2<T>::zero, C2<T>::zero, C2<T>::zero, C2<T>::zero};
        T qR[4] = {C2<T>::zero, C2<T>::zero, C2<T>::zero, C2<T>::zero};
        for (int k = 0; k < nb; ++k) {
            const T b = fbL[(f * nqf + q) * nb + k];
            for (int v = 0; v < 4; ++v) qL[v] += b * coeffs[(iL * 4 + v) * nb + k];
        }
        T zLx[4], zLy[4], zRx[4], zRy[4];
        if (VIS) {
            trace4(fbL + (f * nqf + q) * nb, aux + iL * 8 * nb, nb, zLx);
            trace4(fbL + (f * nqf + q) * nb, aux + (iL * 8 + 4) * nb, nb, zLy);
            for (int v = 0; v < 4; ++v) {
                zRx[v] = zLx[v];
                zRy[v] = zLy[v];
            }
        }
        if (iR >= 0) {
            for (int k = 0; k < nb; ++k) {
                const T b = fbR[(f * nqf + q) * nb + k];
                for (int v = 0; v < 4; ++v) qR[v] += b * coeffs[(iR * 4 + v) * nb + k];
            }
            if (VIS) {
                trace4(fbR + (f * nqf + q) * nb, aux + iR * 8 * nb, nb, zRx);
                trace4(fbR + (f * nqf + q) * nb, aux + (iR * 8 + 4) * nb, nb, zRy);
            }
        } else {
            if (qL[0] <= C2<T>::zero) {
                errf[f] = 1;
                continue;
            }
            T u, v;
            const T pL = prim2(qL[0], qL[1], qL[2], qL[3], g, u, v);
            if (pL <= C2<T>::zero) {
                errf[f] = 1;
                continue;
            }
            const T qf[4] = {qinf[0], qinf[1], qinf[2], qinf[3]};
            bstate2(bc_code[f], qL, nx, ny, qf, g, qR);
        }
        T h[4];
        const bool ok = flux_kind == HODG_FLUX_LLF ? llf2(qL, qR, nx, ny, g, h) : roe2(qL, qR, nx, ny, g, h);
        if (!ok) {
            errf[f] = 1;
            continue;
        }
        for (int v = 0; v < 4; ++v) finv[(f * nqf + q) * 4 + v] = h[v];
        if (VIS) {
            T hL[4], hR[4];
            viscn2(qL, zLx, zLy, nx, ny, g, R, m, pr, hL);
            viscn2(qR, zRx, zRy, nx, ny, g, R, m, pr, hR);
            for (int v = 0; v < 4; ++v) {
                fvis[(f * nqf + q) * 4 + v] = C2<T>::half * (hL[v] + hR[v]);
                fqhat[(f * nqf + q) * 4 + v] = C2<T>::half * (qL[v] + qR[v]);
            }
        }
    }
}

// hodg/dg.py:353-460: thread per cell; products at T, accumulation and the
// mass solve in double; VIS = the ivis == 1 branch
template <typename T, bool VIS>
__global__ void rhs_pass2d(int64_t n_cells, int nb, int nqv, int nqf, int maxf, const T* __restrict__ coeffs,
                           const T* __restrict__ aux, const T* __restrict__ finv, const T* __restrict__ fvis,
                           const T* __restrict__ vol_w, const T* __restrict__ vol_basis,
                           const T* __restrict__ vol_gx, const T* __restrict__ vol_gy,
                           const int8_t* __restrict__ cell_nfaces, const int32_t* __restrict__ cell_faces,
                           const int8_t* __restrict__ cell_fsign, const T* __restrict__ face_w,
                           const T* __restrict__ fbL, const T* __restrict__ fbR, const double* __restrict__ minv64,
                           double gamma, double Rgas, double mu, double Pr, double* __restrict__ res,
                           uint8_t* __restrict__ errc) {
    const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= n_cells) return;
    const T g = T(gamma);
    const T R = T(Rgas), m = T(mu), pr = T(Pr);
    double sc[4 * 6];  // nb <= 6 (order <= 2)
    for (int i = 0; i < 4 * nb; ++i) sc[i] = 0.0;
    const T* cc = coeffs + c * 4 * nb;
    for (int qp = 0; qp < nqv; ++qp) {
        const T w = vol_w[c * nqv + qp];
        if (w == C2<T>::zero) continue;
        T qv[4] = {C2<T>::zero, C2<T>::zero, C2<T>::zero, C2<T>::zero};
        for (int k = 0; k < nb; ++k) {
            const T b = vol_basis[(c * nqv + qp) * nb + k];
            for (int v = 0; v < 4; ++v) qv[v] += b * cc[v * nb + k];
        }
        if (qv[0] <= C2<T>::zero) {
            errc[c] = 1;
            continue;
        }
        T u, vv;
        const T p = prim2(qv[0], qv[1], qv[2], qv[3], g, u, vv);
        if (p <= C2<T>::zero) {
            errc[c] = 1;
            continue;
        }
        T ex[4] = {qv[1], qv[1] * u + p, qv[1] * vv, (qv[3] + p) * u};
        T fy[4] = {qv[2], qv[2] * u, qv[2] * vv + p, (qv[3] + p) * vv};
        if (VIS) {
            T zx[4], zy[4], gr[8], st[5];
            trace4(vol_basis + (c * nqv + qp) * nb, aux + c * 8 * nb, nb, zx);
            trace4(vol_basis + (c * nqv + qp) * nb, aux + (c * 8 + 4) * nb, nb, zy);
            vel_temp_grads2(qv[0], qv[1], qv[2], qv[3], zx, zy, g, R, gr);
            stress_heat2(gr, g, R, m, pr, st);
            ex[1] -= st[0];
            ex[2] -= st[1];
            ex[3] -= gr[0] * st[0] + gr[1] * st[1] - st[3];
            fy[1] -= st[1];
            fy[2] -= st[2];
            fy[3] -= gr[0] * st[1] + gr[1] * st[2] - st[4];
        }
        for (int j = 0; j < nb; ++j) {
            const T gx = w * vol_gx[(c * nqv + qp) * nb + j];
            const T gy = w * vol_gy[(c * nqv + qp) * nb + j];
            for (int v = 0; v < 4; ++v) sc[v * nb + j] += ex[v] * gx + fy[v] * gy;
        }
    }
    for (int slot = 0; slot < cell_nfaces[c]; ++slot) {
        const int64_t fid = cell_faces[c * maxf + slot];
        const int sgn = cell_fsign[c * maxf + slot];
        const T* tb = sgn > 0 ? fbL : fbR;
        const T s = T(sgn);
        for (int q = 0; q < nqf; ++q) {
            const T w = s * face_w[fid * nqf + q];
            T h[4];
            for (int v = 0; v < 4; ++v) h[v] = finv[(fid * nqf + q) * 4 + v];
            if (VIS)
                for (int v = 0; v < 4; ++v) h[v] -= fvis[(fid * nqf + q) * 4 + v];
            for (int j = 0; j < nb; ++j) {
                const T wb = w * tb[(fid * nqf + q) * nb + j];
                for (int v = 0; v < 4; ++v) sc[v * nb + j] -= h[v] * wb;
            }
        }
    }
    const double* mi = minv64 + c * nb * nb;
    for (int v = 0; v < 4; ++v)
        for (int j = 0; j < nb; ++j) {
            double acc = 0.0;
            for (int k = 0; k < nb; ++k) acc += mi[j * nb + k] * sc[v * nb + k];
            res[(c * 4 + v) * nb + j] = acc;
        }
}

// hodg/timestepping.py:105-134
template <typename T>
__global__ void dt_pass2d(int64_t n_cells, int nb, const T* __restrict__ coeffs, const double* __restrict__ bmean,
                          const double* __restrict__ h, double gamma, double mu, double cfl, int order,
                          double* __restrict__ out, uint8_t* __restrict__ errc) {
    const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= n_cells) return;
    const double fac = 2.0 * order + 1.0;
    double m[4] = {0.0, 0.0, 0.0, 0.0};
    for (int j = 0; j < nb; ++j) {
        const double b = bmean[c * nb + j];
        for (int v = 0; v < 4; ++v) m[v] += b * double(coeffs[(c * 4 + v) * nb + j]);
    }
    if (m[0] <= 0.0) {
        errc[c] = 1;
        out[c] = 0.0;
        return;
    }
    const double u = m[1] / m[0], v = m[2] / m[0];
    const double p = (gamma - 1.0) * (m[3] - 0.5 * m[0] * (u * u + v * v));
    if (p <= 0.0) {
        errc[c] = 1;
        out[c] = 0.0;
        return;
    }
    const double a = sqrt(gamma * p / m[0]);
    const double speed = sqrt(u * u + v * v) + a + 2.0 * mu * fac / (m[0] * h[c]);
    out[c] = cfl * h[c] / (fac * speed);
}

// hodg/timestepping.py:165-180
template <typename T>
__global__ void axpy2d(int64_t n, int per, const T* __restrict__ u, const double* __restrict__ r,
                       const double* __restrict__ dtc, T* __restrict__ out) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n * per) return;
    out[k] = T(double(u[k]) + dtc[k / per] * r[k]);
}

template <typename T>
__global__ void combine2d(int64_t n, int per, const T* __restrict__ u, const T* __restrict__ u1,
                          const double* __restrict__ r1, const double* __restrict__ dtc, T* __restrict__ out) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n * per) return;
    const T s = u[k] + u1[k];
    out[k] = T(0.5 * (double(s) + dtc[k / per] * r1[k]));
}

inline unsigned nblk(int64_t n) { return unsigned((n + 127) / 128); }
inline int rc() { return cudaGetLastError() == cudaSuccess ? HODG_OK : HODG_ECUDA; }

template <bool VIS>
int flux2d_dispatch(int prec, int64_t n_faces, int nqf, int nb, const void* coeffs, const void* aux, const void* fbL,
                    const void* fbR, const int32_t* face_cells, const int8_t* bc_code, const void* fnx,
                    const void* fny, const void* qinf, double gamma, double Rgas, double mu, double Pr, int flux_kind,
                    void* finv, void* fvis, void* fqhat, uint8_t* errf, void* stream) {
    if (n_faces <= 0 || nb < 1 || nb > 6 || nqf < 1) return HODG_EINVAL;
    hodg_count_launch(1);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
#define HODG_FLUX_ARGS(T)                                                                                            \
    n_faces, nqf, nb, (const T*)coeffs, (const T*)aux, (const T*)fbL, (const T*)fbR, face_cells, bc_code,           \
        (const T*)fnx, (const T*)fny, (const T*)qinf, gamma, Rgas, mu, Pr, flux_kind, (T*)finv, (T*)fvis, (T*)fqhat, \
        errf
    if (prec == HODG_PREC_F64)
        flux_pass2d<double, VIS><<<nblk(n_faces), 128, 0, st>>>(HODG_FLUX_ARGS(double));
    else
        flux_pass2d<float, VIS><<<nblk(n_faces), 128, 0, st>>>(HODG_FLUX_ARGS(float));
#undef HODG_FLUX_ARGS
    return rc();
}

template <bool VIS>
int rhs2d_dispatch(int prec, int64_t n_cells, int nb, int nqv, int nqf, int maxf, const void* coeffs,
                   const void* aux, const void* finv, const void* fvis, const void* vol_w, const void* vol_basis,
                   const void* vol_gx, const void* vol_gy, const int8_t* cell_nfaces, const int32_t* cell_faces,
                   const int8_t* cell_fsign, const void* face_w, const void* fbL, const void* fbR,
                   const double* minv64, double gamma, double Rgas, double mu, double Pr, double* res, uint8_t* errc,
                   void* stream) {
    if (n_cells <= 0 || nb < 1 || nb > 6) return HODG_EINVAL;
    hodg_count_launch(1);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
#define HODG_RHS_ARGS(T)                                                                                             \
    n_cells, nb, nqv, nqf, maxf, (const T*)coeffs, (const T*)aux, (const T*)finv, (const T*)fvis, (const T*)vol_w,   \
        (const T*)vol_basis, (const T*)vol_gx, (const T*)vol_gy, cell_nfaces, cell_faces, cell_fsign,               \
        (const T*)face_w, (const T*)fbL, (const T*)fbR, minv64, gamma, Rgas, mu, Pr, res, errc
    if (prec == HODG_PREC_F64)
        rhs_pass2d<double, VIS><<<nblk(n_cells), 128, 0, st>>>(HODG_RHS_ARGS(double));
    else
        rhs_pass2d<float, VIS><<<nblk(n_cells), 128, 0, st>>>(HODG_RHS_ARGS(float));
#undef HODG_RHS_ARGS
    return rc();
}

}  // namespace

extern "C" {

int hodg2d_flux_pass(int prec, int64_t n_faces, int nqf, int nb, const void* coeffs, const void* fbL, const void* fbR,
                     const int32_t* face_cells, const int8_t* bc_code, const void* fnx, const void* fny,
                     const void* qinf, double gamma, int flux_kind, void* finv, uint8_t* errf, void* stream) {
    return flux2d_dispatch<false>(prec, n_faces, nqf, nb, coeffs, nullptr, fbL, fbR, face_cells, bc_code, fnx, fny,
                                  qinf, gamma, 1.0, 0.0, 1.0, flux_kind, finv, nullptr, nullptr, errf, stream);
}

int hodg2d_flux_pass_ns(int prec, int64_t n_faces, int nqf, int nb, const void* coeffs, const void* aux,
                        const void* fbL, const void* fbR, const int32_t* face_cells, const int8_t* bc_code,
                        const void* fnx, const void* fny, const void* qinf, double gamma, double Rgas, double mu,
                        double Pr, void* finv, void* fvis, void* fqhat, uint8_t* errf, void* stream) {
    if (aux == nullptr || fvis == nullptr || fqhat == nullptr) return HODG_EINVAL;
    return flux2d_dispatch<true>(prec, n_faces, nqf, nb, coeffs, aux, fbL, fbR, face_cells, bc_code, fnx, fny, qinf,
                                 gamma, Rgas, mu, Pr, HODG_FLUX_ROE, finv, fvis, fqhat, errf, stream);
}

int hodg2d_rhs_pass(int prec, int64_t n_cells, int nb, int nqv, int nqf, int maxf, const void* coeffs,
                    const void* finv, const void* vol_w, const void* vol_basis, const void* vol_gx,
                    const void* vol_gy, const int8_t* cell_nfaces, const int32_t* cell_faces,
                    const int8_t* cell_fsign, const void* face_w, const void* fbL, const void* fbR,
                    const double* minv64, double gamma, double* res, uint8_t* errc, void* stream) {
    return rhs2d_dispatch<false>(prec, n_cells, nb, nqv, nqf, maxf, coeffs, nullptr, finv, nullptr, vol_w, vol_basis,
                                 vol_gx, vol_gy, cell_nfaces, cell_faces, cell_fsign, face_w, fbL, fbR, minv64, gamma,
                                 1.0, 0.0, 1.0, res, errc, stream);
}

int hodg2d_rhs_pass_ns(int prec, int64_t n_cells, int nb, int nqv, int nqf, int maxf, const void* coeffs,
                       const void* aux, const void* finv, const void* fvis, const void* vol_w, const void* vol_basis,
                       const void* vol_gx, const void* vol_gy, const int8_t* cell_nfaces, const int32_t* cell_faces,
                       const int8_t* cell_fsign, const void* face_w, const void* fbL, const void* fbR,
                       const double* minv64, double gamma, double Rgas, double mu, double Pr, double* res,
                       uint8_t* errc, void* stream) {
    if (aux == nullptr || fvis == nullptr) return HODG_EINVAL;
    return rhs2d_dispatch<true>(prec, n_cells, nb, nqv, nqf, maxf, coeffs, aux, finv, fvis, vol_w, vol_basis, vol_gx,
                                vol_gy, cell_nfaces, cell_faces, cell_fsign, face_w, fbL, fbR, minv64, gamma, Rgas,
                                mu, Pr, res, errc, stream);
}

int hodg2d_qhat_pass(int prec, int64_t n_faces, int nqf, int nb, const void* coeffs, const void* fbL, const void* fbR,
                     const int32_t* face_cells, const int8_t* bc_code, const void* fnx, const void* fny,
                     const void* qinf, double gamma, void* qhat, uint8_t* errf, void* stream) {
    if (n_faces <= 0 || nb < 1 || nb > 6 || nqf < 1) return HODG_EINVAL;
    hodg_count_launch(1);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (prec == HODG_PREC_F64)
        qhat_pass2d<double><<<nblk(n_faces), 128, 0, st>>>(
            n_faces, nqf, nb, (const double*)coeffs, (const double*)fbL, (const double*)fbR, face_cells, bc_code,
            (const double*)fnx, (const double*)fny, (const double*)qinf, gamma, (double*)qhat, errf);
    else
        qhat_pass2d<float><<<nblk(n_faces), 128, 0, st>>>(
            n_faces, nqf, nb, (const float*)coeffs, (const float*)fbL, (const float*)fbR, face_cells, bc_code,
            (const float*)fnx, (const float*)fny, (const float*)qinf, gamma, (float*)qhat, errf);
    return rc();
}

int hodg2d_aux_pass(int prec, int64_t n_cells, int nb, int nqv, int nqf, int maxf, const void* coeffs,
                    const void* qhat, const void* vol_w, const void* vol_basis, const void* vol_gx,
                    const void* vol_gy, const int8_t* cell_nfaces, const int32_t* cell_faces,
                    const int8_t* cell_fsign, const void* face_w, const void* fbL, const void* fbR, const void* fnx,
                    const void* fny, const void* minv, void* aux, void* stream) {
    if (n_cells <= 0 || nb < 1 || nb > 6) return HODG_EINVAL;
    hodg_count_launch(1);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
#define HODG_AUX_ARGS(T)                                                                                             \
    n_cells, nb, nqv, nqf, maxf, (const T*)coeffs, (const T*)qhat, (const T*)vol_w, (const T*)vol_basis,             \
        (const T*)vol_gx, (const T*)vol_gy, cell_nfaces, cell_faces, cell_fsign, (const T*)face_w, (const T*)fbL,    \
        (const T*)fbR, (const T*)fnx, (const T*)fny, (const T*)minv, (T*)aux
    if (prec == HODG_PREC_F64)
        aux_pass2d<double><<<nblk(n_cells), 128, 0, st>>>(HODG_AUX_ARGS(double));
    else
        aux_pass2d<float><<<nblk(n_cells), 128, 0, st>>>(HODG_AUX_ARGS(float));
#undef HODG_AUX_ARGS
    return rc();
}

int hodg2d_dt_pass(int prec, int64_t n_cells, int nb, const void* coeffs, const double* basis_mean, const double* h,
                   double gamma, double mu, double cfl, int order, double* out, uint8_t* errc, void* stream) {
    if (n_cells <= 0) return HODG_EINVAL;
    hodg_count_launch(1);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (prec == HODG_PREC_F64)
        dt_pass2d<double><<<nblk(n_cells), 128, 0, st>>>(n_cells, nb, (const double*)coeffs, basis_mean, h, gamma,
                                                          mu, cfl, order, out, errc);
    else
        dt_pass2d<float><<<nblk(n_cells), 128, 0, st>>>(n_cells, nb, (const float*)coeffs, basis_mean, h, gamma, mu,
                                                         cfl, order, out, errc);
    return rc();
}

int hodg2d_axpy(int prec, int64_t n_cells, int per_cell, const void* u, const double* r, const double* dtc, void* out,
                void* stream) {
    hodg_count_launch(1);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (prec == HODG_PREC_F64)
        axpy2d<double><<<nblk(n_cells * per_cell), 128, 0, st>>>(n_cells, per_cell, (const double*)u, r, dtc,
                                                                  (double*)out);
    else
        axpy2d<float><<<nblk(n_cells * per_cell), 128, 0, st>>>(n_cells, per_cell, (const float*)u, r, dtc,
                                                                 (float*)out);
    return rc();
}

int hodg2d_combine(int prec, int64_t n_cells, int per_cell, const void* u, const void* u1, const double* r1,
                   const double* dtc, void* out, void* stream) {
    hodg_count_launch(1);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (prec == HODG_PREC_F64)
        combine2d<double><<<nblk(n_cells * per_cell), 128, 0, st>>>(n_cells, per_cell, (const double*)u,
                                                                     (const double*)u1, r1, dtc, (double*)out);
    else
        combine2d<float><<<nblk(n_cells * per_cell), 128, 0, st>>>(n_cells, per_cell, (const float*)u,
                                                                    (const float*)u1, r1, dtc, (float*)out);
    return rc();
}

}  // extern "C"
