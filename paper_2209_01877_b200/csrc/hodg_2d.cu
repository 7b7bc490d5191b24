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
            s = pi / pow(rho, g);
            utx = ui - uni * nx;
            uty = vi - uni * ny;
        } else {
            s = pf / pow(rf, g);
            utx = uf - unf * nx;
            uty = vf - unf * ny;
        }
        const T rb = pow(ab * ab / (g * s), one / (g - one));
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

// hodg/dg.py:240-351 (Euler branch): thread per face
template <typename T>
__global__ void flux_pass2d(int64_t n_faces, int nqf, int nb, const T* __restrict__ coeffs, const T* __restrict__ fbL,
                            const T* __restrict__ fbR, const int32_t* __restrict__ face_cells,
                            const int8_t* __restrict__ bc_code, const T* __restrict__ fnx, const T* __restrict__ fny,
                            const T* __restrict__ qinf, double gamma, int flux_kind, T* __restrict__ finv,
                            uint8_t* __restrict__ errf) {
    const int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (f >= n_faces) return;
    const T g = T(gamma);
    const int64_t iL = face_cells[2 * f], iR = face_cells[2 * f + 1];
    const T nx = fnx[f], ny = fny[f];
    for (int q = 0; q < nqf; ++q) {
        T qL[4] = {C2<T>::zero, C2<T>::zero, C2<T>::zero, C2<T>::zero};
        T qR[4] = {C2<T>::zero, C2<T>::zero, C2<T>::zero, C2<T>::zero};
        for (int k = 0; k < nb; ++k) {
            const T b = fbL[(f * nqf + q) * nb + k];
            for (int v = 0; v < 4; ++v) qL[v] += b * coeffs[(iL * 4 + v) * nb + k];
        }
        if (iR >= 0) {
            for (int k = 0; k < nb; ++k) {
                const T b = fbR[(f * nqf + q) * nb + k];
                for (int v = 0; v < 4; ++v) qR[v] += b * coeffs[(iR * 4 + v) * nb + k];
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
    }
}

// hodg/dg.py:353-460 (Euler branch): thread per cell; products at T,
// accumulation and the mass solve in double
template <typename T>
__global__ void rhs_pass2d(int64_t n_cells, int nb, int nqv, int nqf, int maxf, const T* __restrict__ coeffs,
                           const T* __restrict__ finv, const T* __restrict__ vol_w, const T* __restrict__ vol_basis,
                           const T* __restrict__ vol_gx, const T* __restrict__ vol_gy,
                           const int8_t* __restrict__ cell_nfaces, const int32_t* __restrict__ cell_faces,
                           const int8_t* __restrict__ cell_fsign, const T* __restrict__ face_w,
                           const T* __restrict__ fbL, const T* __restrict__ fbR, const double* __restrict__ minv64,
                           double gamma, double* __restrict__ res, uint8_t* __restrict__ errc) {
    const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= n_cells) return;
    const T g = T(gamma);
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
        const T ex[4] = {qv[1], qv[1] * u + p, qv[1] * vv, (qv[3] + p) * u};
        const T fy[4] = {qv[2], qv[2] * u, qv[2] * vv + p, (qv[3] + p) * vv};
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
            const T* h = finv + (fid * nqf + q) * 4;
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

}  // namespace

extern int64_t hodg_count_launch(int64_t n);

extern "C" {

int hodg2d_flux_pass(int prec, int64_t n_faces, int nqf, int nb, const void* coeffs, const void* fbL, const void* fbR,
                     const int32_t* face_cells, const int8_t* bc_code, const void* fnx, const void* fny,
                     const void* qinf, double gamma, int flux_kind, void* finv, uint8_t* errf, void* stream) {
    if (n_faces <= 0 || nb < 1 || nb > 6 || nqf < 1) return HODG_EINVAL;
    hodg_count_launch(1);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (prec == HODG_PREC_F64)
        flux_pass2d<double><<<nblk(n_faces), 128, 0, st>>>(
            n_faces, nqf, nb, (const double*)coeffs, (const double*)fbL, (const double*)fbR, face_cells, bc_code,
            (const double*)fnx, (const double*)fny, (const double*)qinf, gamma, flux_kind, (double*)finv, errf);
    else
        flux_pass2d<float><<<nblk(n_faces), 128, 0, st>>>(
            n_faces, nqf, nb, (const float*)coeffs, (const float*)fbL, (const float*)fbR, face_cells, bc_code,
            (const float*)fnx, (const float*)fny, (const float*)qinf, gamma, flux_kind, (float*)finv, errf);
    return rc();
}

int hodg2d_rhs_pass(int prec, int64_t n_cells, int nb, int nqv, int nqf, int maxf, const void* coeffs,
                    const void* finv, const void* vol_w, const void* vol_basis, const void* vol_gx,
                    const void* vol_gy, const int8_t* cell_nfaces, const int32_t* cell_faces,
                    const int8_t* cell_fsign, const void* face_w, const void* fbL, const void* fbR,
                    const double* minv64, double gamma, double* res, uint8_t* errc, void* stream) {
    if (n_cells <= 0 || nb < 1 || nb > 6) return HODG_EINVAL;
    hodg_count_launch(1);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (prec == HODG_PREC_F64)
        rhs_pass2d<double><<<nblk(n_cells), 128, 0, st>>>(
            n_cells, nb, nqv, nqf, maxf, (const double*)coeffs, (const double*)finv, (const double*)vol_w,
            (const double*)vol_basis, (const double*)vol_gx, (const double*)vol_gy, cell_nfaces, cell_faces,
            cell_fsign, (const double*)face_w, (const double*)fbL, (const double*)fbR, minv64, gamma, res, errc);
    else
        rhs_pass2d<float><<<nblk(n_cells), 128, 0, st>>>(
            n_cells, nb, nqv, nqf, maxf, (const float*)coeffs, (const float*)finv, (const float*)vol_w,
            (const float*)vol_basis, (const float*)vol_gx, (const float*)vol_gy, cell_nfaces, cell_faces,
            cell_fsign, (const float*)face_w, (const float*)fbL, (const float*)fbR, minv64, gamma, res, errc);
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
