/* Body of the CPU oracle kernels, included once per precision by
 * hodg_oracle.c with REAL / SFX defined.  TEST INFRASTRUCTURE ONLY: this is
 * the checker the CUDA path is compared against, never the product.
 *
 * Each function restates one numba kernel of the reference with the same
 * loop order and the same expression trees (no FMA contraction: built with
 * -ffp-contract=off), so in 2D the results are bitwise equal to the
 * reference's LLVM code.  The 3D (tetrahedral, 5-variable) branches extend
 * the same formulas with the z components; every such extension is guarded
 * by `d3` so the 2D expression trees are untouched.
 */

#define ONE ((REAL)1.0)
#define ZERO ((REAL)0.0)
#define HALF ((REAL)0.5)
#define TWO ((REAL)2.0)
#define QUARTER ((REAL)0.25)
#define EFIX ((REAL)0.05)

/* hodg/physics.py:159-165 (prim) generalised to 3D; returns p */
static inline REAL CAT(prim_p, SFX)(REAL rho, REAL ru, REAL rv, REAL rw, REAL e, REAL g,
                                    int d3, REAL *u, REAL *v, REAL *w) {
    *u = ru / rho;
    *v = rv / rho;
    if (d3) {
        *w = rw / rho;
        return (g - ONE) * (e - HALF * rho * (*u * *u + *v * *v + *w * *w));
    }
    *w = ZERO;
    return (g - ONE) * (e - HALF * rho * (*u * *u + *v * *v));
}

/* hodg/physics.py:168-169 (energy) */
static inline REAL CAT(energy, SFX)(REAL rho, REAL u, REAL v, REAL w, REAL p, REAL g, int d3) {
    if (d3) return p / (g - ONE) + HALF * rho * (u * u + v * v + w * w);
    return p / (g - ONE) + HALF * rho * (u * u + v * v);
}

/* Unpack / pack helpers: q[] is (rho, ru, rv, [rw,] e). */
#define QE(q) ((q)[d3 ? 4 : 3])

/* hodg/physics.py:177-250 (roe), 3D extension: extra shear wave in the l2
 * family.  Returns ok (0 on inadmissible input or failed Roe average). */
static int CAT(roe, SFX)(const REAL *qL, const REAL *qR, const REAL *n, REAL g, int d3, REAL *f) {
    REAL rL = qL[0], rR = qR[0];
    if (rL <= ZERO || rR <= ZERO) return 0;
    REAL ruL = qL[1], rvL = qL[2], rwL = d3 ? qL[3] : ZERO, eL = QE(qL);
    REAL ruR = qR[1], rvR = qR[2], rwR = d3 ? qR[3] : ZERO, eR = QE(qR);
    REAL uL, vL, wL, uR, vR, wR;
    REAL pL = CAT(prim_p, SFX)(rL, ruL, rvL, rwL, eL, g, d3, &uL, &vL, &wL);
    REAL pR = CAT(prim_p, SFX)(rR, ruR, rvR, rwR, eR, g, d3, &uR, &vR, &wR);
    if (pL <= ZERO || pR <= ZERO) return 0;
    REAL nx = n[0], ny = n[1], nz = d3 ? n[2] : ZERO;

    /* fluxn (hodg/physics.py:172-175) */
    REAL vnL = d3 ? uL * nx + vL * ny + wL * nz : uL * nx + vL * ny;
    REAL vnR = d3 ? uR * nx + vR * ny + wR * nz : uR * nx + vR * ny;
    REAL fL0 = rL * vnL, fL1 = ruL * vnL + pL * nx, fL2 = rvL * vnL + pL * ny;
    REAL fL3 = d3 ? rwL * vnL + pL * nz : ZERO, fLE = (eL + pL) * vnL;
    REAL fR0 = rR * vnR, fR1 = ruR * vnR + pR * nx, fR2 = rvR * vnR + pR * ny;
    REAL fR3 = d3 ? rwR * vnR + pR * nz : ZERO, fRE = (eR + pR) * vnR;

    REAL sL = SQRT(rL);
    REAL sR = SQRT(rR);
    REAL den = sL + sR;
    REAL ut = (sL * uL + sR * uR) / den;
    REAL vt = (sL * vL + sR * vR) / den;
    REAL wt = d3 ? (sL * wL + sR * wR) / den : ZERO;
    REAL HL = (eL + pL) / rL;
    REAL HR = (eR + pR) / rR;
    REAL Ht = (sL * HL + sR * HR) / den;
    REAL ke = d3 ? HALF * (ut * ut + vt * vt + wt * wt) : HALF * (ut * ut + vt * vt);
    REAL a2 = (g - ONE) * (Ht - ke);
    if (a2 <= ZERO) return 0;
    REAL a = SQRT(a2);
    REAL rt = sL * sR;
    REAL unt = d3 ? ut * nx + vt * ny + wt * nz : ut * nx + vt * ny;

    REAL dr = rR - rL;
    REAL dp = pR - pL;
    REAL du = uR - uL;
    REAL dv = vR - vL;
    REAL dw = d3 ? wR - wL : ZERO;
    REAL dun = d3 ? (uR * nx + vR * ny + wR * nz) - (uL * nx + vL * ny + wL * nz)
                  : (uR * nx + vR * ny) - (uL * nx + vL * ny);

    REAL l1 = FABS(unt - a);
    REAL l2 = FABS(unt);
    REAL l4 = FABS(unt + a);
    REAL delta = EFIX * a;
    if (l1 < delta) l1 = HALF * (l1 * l1 / delta + delta);
    if (l4 < delta) l4 = HALF * (l4 * l4 / delta + delta);

    REAL a1 = (dp - rt * a * dun) / (TWO * a2);
    REAL a4 = (dp + rt * a * dun) / (TWO * a2);
    REAL a2w = dr - dp / a2;

    REAL d0 = l1 * a1 + l2 * a2w + l4 * a4;
    REAL d1 = l1 * a1 * (ut - a * nx) + l2 * (a2w * ut + rt * (du - dun * nx)) + l4 * a4 * (ut + a * nx);
    REAL d2 = l1 * a1 * (vt - a * ny) + l2 * (a2w * vt + rt * (dv - dun * ny)) + l4 * a4 * (vt + a * ny);
    REAL d3w = d3 ? l1 * a1 * (wt - a * nz) + l2 * (a2w * wt + rt * (dw - dun * nz)) + l4 * a4 * (wt + a * nz)
                  : ZERO;
    REAL dE = d3 ? l1 * a1 * (Ht - a * unt) +
                       l2 * (a2w * ke + rt * (ut * du + vt * dv + wt * dw - unt * dun)) +
                       l4 * a4 * (Ht + a * unt)
                 : l1 * a1 * (Ht - a * unt) + l2 * (a2w * ke + rt * (ut * du + vt * dv - unt * dun)) +
                       l4 * a4 * (Ht + a * unt);
    f[0] = HALF * (fL0 + fR0) - HALF * d0;
    f[1] = HALF * (fL1 + fR1) - HALF * d1;
    f[2] = HALF * (fL2 + fR2) - HALF * d2;
    if (d3) {
        f[3] = HALF * (fL3 + fR3) - HALF * d3w;
        f[4] = HALF * (fLE + fRE) - HALF * dE;
    } else {
        f[3] = HALF * (fLE + fRE) - HALF * dE;
    }
    return 1;
}

/* Local Lax-Friedrichs (Rusanov) flux: north_star's alternative to Roe; not
 * in the reference.  F = (F_L + F_R)/2 - lambda/2 (q_R - q_L),
 * lambda = max(|u_n| + a) over both sides. */
static int CAT(llf, SFX)(const REAL *qL, const REAL *qR, const REAL *n, REAL g, int d3, REAL *f) {
    REAL rL = qL[0], rR = qR[0];
    if (rL <= ZERO || rR <= ZERO) return 0;
    REAL uL, vL, wL, uR, vR, wR;
    REAL pL = CAT(prim_p, SFX)(rL, qL[1], qL[2], d3 ? qL[3] : ZERO, QE(qL), g, d3, &uL, &vL, &wL);
    REAL pR = CAT(prim_p, SFX)(rR, qR[1], qR[2], d3 ? qR[3] : ZERO, QE(qR), g, d3, &uR, &vR, &wR);
    if (pL <= ZERO || pR <= ZERO) return 0;
    REAL nx = n[0], ny = n[1], nz = d3 ? n[2] : ZERO;
    REAL vnL = d3 ? uL * nx + vL * ny + wL * nz : uL * nx + vL * ny;
    REAL vnR = d3 ? uR * nx + vR * ny + wR * nz : uR * nx + vR * ny;
    REAL aL = SQRT(g * pL / rL);
    REAL aR = SQRT(g * pR / rR);
    REAL sl = FABS(vnL) + aL;
    REAL sr = FABS(vnR) + aR;
    REAL lam = sl > sr ? sl : sr;
    REAL FL[5], FR[5];
    int nv = d3 ? 5 : 4;
    FL[0] = rL * vnL;
    FL[1] = qL[1] * vnL + pL * nx;
    FL[2] = qL[2] * vnL + pL * ny;
    FR[0] = rR * vnR;
    FR[1] = qR[1] * vnR + pR * nx;
    FR[2] = qR[2] * vnR + pR * ny;
    if (d3) {
        FL[3] = qL[3] * vnL + pL * nz;
        FR[3] = qR[3] * vnR + pR * nz;
    }
    FL[nv - 1] = (QE(qL) + pL) * vnL;
    FR[nv - 1] = (QE(qR) + pR) * vnR;
    for (int v = 0; v < nv; ++v) f[v] = HALF * (FL[v] + FR[v]) - HALF * lam * (qR[v] - qL[v]);
    return 1;
}

/* hodg/physics.py:292-344 (bstate_slip / bstate_noslip / bstate_far /
 * boundary), 3D extension: tangential velocity is a 3-vector. */
static void CAT(bstate, SFX)(int kind, const REAL *q, const REAL *n, const REAL *qf, REAL g, int d3,
                             REAL *out) {
    int nv = d3 ? 5 : 4;
    REAL nx = n[0], ny = n[1], nz = d3 ? n[2] : ZERO;
    if (kind == 1) {
        REAL rho = q[0], ru = q[1], rv = q[2], rw = d3 ? q[3] : ZERO, e = QE(q);
        REAL rf = qf[0], ruf = qf[1], rvf = qf[2], rwf = d3 ? qf[3] : ZERO, ef = QE(qf);
        REAL ui, vi, wi, uf, vf, wf;
        REAL pi = CAT(prim_p, SFX)(rho, ru, rv, rw, e, g, d3, &ui, &vi, &wi);
        REAL pf = CAT(prim_p, SFX)(rf, ruf, rvf, rwf, ef, g, d3, &uf, &vf, &wf);
        REAL ai = SQRT(g * pi / rho);
        REAL af = SQRT(g * pf / rf);
        REAL uni = d3 ? ui * nx + vi * ny + wi * nz : ui * nx + vi * ny;
        REAL unf = d3 ? uf * nx + vf * ny + wf * nz : uf * nx + vf * ny;
        if (uni >= ai) {
            for (int v = 0; v < nv; ++v) out[v] = q[v];
            return;
        }
        if (unf <= -af) {
            for (int v = 0; v < nv; ++v) out[v] = qf[v];
            return;
        }
        REAL rplus = uni + TWO * ai / (g - ONE);
        REAL rminus = unf - TWO * af / (g - ONE);
        REAL unb = HALF * (rplus + rminus);
        REAL ab = QUARTER * (g - ONE) * (rplus - rminus);
        if (!(ab > ZERO)) {
            for (int v = 0; v < nv; ++v) out[v] = qf[v];
            return;
        }
        REAL s, utx, uty, utz;
        if (unb > ZERO) {
            s = pi / POW(rho, g);
            utx = ui - uni * nx;
            uty = vi - uni * ny;
            utz = d3 ? wi - uni * nz : ZERO;
        } else {
            s = pf / POW(rf, g);
            utx = uf - unf * nx;
            uty = vf - unf * ny;
            utz = d3 ? wf - unf * nz : ZERO;
        }
        REAL rb = POW(ab * ab / (g * s), ONE / (g - ONE));
        REAL pb = rb * ab * ab / g;
        REAL ub = utx + unb * nx;
        REAL vb = uty + unb * ny;
        REAL wb = d3 ? utz + unb * nz : ZERO;
        out[0] = rb;
        out[1] = rb * ub;
        out[2] = rb * vb;
        if (d3) out[3] = rb * wb;
        out[nv - 1] = CAT(energy, SFX)(rb, ub, vb, wb, pb, g, d3);
    } else if (kind == 2) {
        REAL un2 = d3 ? TWO * (q[1] * nx + q[2] * ny + q[3] * nz) : TWO * (q[1] * nx + q[2] * ny);
        out[0] = q[0];
        out[1] = q[1] - un2 * nx;
        out[2] = q[2] - un2 * ny;
        if (d3) out[3] = q[3] - un2 * nz;
        out[nv - 1] = q[nv - 1];
    } else {
        out[0] = q[0];
        out[1] = -q[1];
        out[2] = -q[2];
        if (d3) out[3] = -q[3];
        out[nv - 1] = q[nv - 1];
    }
}

/* ---- viscous (BR1) terms, 2D: hodg/physics.py:252-290, hodg/dg.py:114-238 ---- */

/* hodg/physics.py:252-269 */
static inline void CAT(vel_temp_grads, SFX)(REAL rho, REAL ru, REAL rv, REAL e, const REAL *zx, const REAL *zy,
                                            REAL gamma, REAL Rgas, REAL *out8) {
    REAL u = ru / rho;
    REAL v = rv / rho;
    REAL ux = (zx[1] - u * zx[0]) / rho;
    REAL vx = (zx[2] - v * zx[0]) / rho;
    REAL uy = (zy[1] - u * zy[0]) / rho;
    REAL vy = (zy[2] - v * zy[0]) / rho;
    REAL ke = HALF * (u * u + v * v);
    REAL ein = e - rho * ke;
    REAL kx = ke * zx[0] + rho * (u * ux + v * vx);
    REAL ky = ke * zy[0] + rho * (u * uy + v * vy);
    REAL coef = (gamma - ONE) / Rgas;
    REAL Tx = coef * ((zx[3] - kx) * rho - ein * zx[0]) / (rho * rho);
    REAL Ty = coef * ((zy[3] - ky) * rho - ein * zy[0]) / (rho * rho);
    out8[0] = u; out8[1] = v; out8[2] = ux; out8[3] = uy; out8[4] = vx; out8[5] = vy; out8[6] = Tx; out8[7] = Ty;
}

/* hodg/physics.py:271-277; returns txx, txy, tyy, qx, qy */
static inline void CAT(stress_heat, SFX)(REAL ux, REAL uy, REAL vx, REAL vy, REAL Tx, REAL Ty, REAL gamma,
                                         REAL Rgas, REAL mu, REAL Pr, REAL *o5) {
    const REAL two_thirds = (REAL)(2.0 / 3.0);
    o5[0] = mu * two_thirds * (TWO * ux - vy);
    o5[2] = mu * two_thirds * (TWO * vy - ux);
    o5[1] = mu * (uy + vx);
    REAL k = mu * gamma * Rgas / ((gamma - ONE) * Pr);
    o5[3] = -k * Tx;
    o5[4] = -k * Ty;
}

/* hodg/physics.py:279-290 */
static inline void CAT(viscn, SFX)(REAL rho, REAL ru, REAL rv, REAL e, const REAL *zx, const REAL *zy, REAL nx,
                                   REAL ny, REAL gamma, REAL Rgas, REAL mu, REAL Pr, REAL *h) {
    REAL g8[8], s5[5];
    CAT(vel_temp_grads, SFX)(rho, ru, rv, e, zx, zy, gamma, Rgas, g8);
    CAT(stress_heat, SFX)(g8[2], g8[3], g8[4], g8[5], g8[6], g8[7], gamma, Rgas, mu, Pr, s5);
    REAL u = g8[0], v = g8[1];
    h[0] = ZERO;
    h[1] = s5[0] * nx + s5[1] * ny;
    h[2] = s5[1] * nx + s5[2] * ny;
    h[3] = (u * s5[0] + v * s5[1] - s5[3]) * nx + (u * s5[1] + v * s5[2] - s5[4]) * ny;
}

/* hodg/dg.py:114-162 (qhat_pass): central trace average; 2D */
void CAT(ora_qhat_pass, SFX)(int64_t n_faces, int nqf, int nb, const REAL *coeffs, const REAL *fbL, const REAL *fbR,
                             const int32_t *face_cells, const int8_t *bc_code, const REAL *fnx, const REAL *fny,
                             const REAL *qinf, double gamma, REAL *qhat, uint8_t *errf) {
    const int d3 = 0;
    const REAL g = (REAL)gamma;
#pragma omp parallel for schedule(static)
    for (int64_t f = 0; f < n_faces; ++f) {
        int64_t iL = face_cells[2 * f], iR = face_cells[2 * f + 1];
        REAL n[2] = {fnx[f], fny[f]};
        for (int q = 0; q < nqf; ++q) {
            REAL qL[4] = {ZERO, ZERO, ZERO, ZERO}, qR[4] = {ZERO, ZERO, ZERO, ZERO};
            for (int k = 0; k < nb; ++k) {
                REAL b = fbL[(f * nqf + q) * nb + k];
                for (int v = 0; v < 4; ++v) qL[v] += b * coeffs[(iL * 4 + v) * nb + k];
            }
            if (iR >= 0) {
                for (int k = 0; k < nb; ++k) {
                    REAL b = fbR[(f * nqf + q) * nb + k];
                    for (int v = 0; v < 4; ++v) qR[v] += b * coeffs[(iR * 4 + v) * nb + k];
                }
            } else {
                if (qL[0] <= ZERO) {
                    errf[f] = 1;
                    continue;
                }
                REAL u, v, w;
                REAL pL = CAT(prim_p, SFX)(qL[0], qL[1], qL[2], ZERO, qL[3], g, d3, &u, &v, &w);
                if (pL <= ZERO) {
                    errf[f] = 1;
                    continue;
                }
                CAT(bstate, SFX)(bc_code[f], qL, n, qinf, g, d3, qR);
            }
            for (int v = 0; v < 4; ++v) qhat[(f * nqf + q) * 4 + v] = HALF * (qL[v] + qR[v]);
        }
    }
}

/* hodg/dg.py:164-238 (aux_pass): weak gradient z = M^-1 [-int Q grad b + sum qhat n b] (2D).
 * aux is (N, 2, 4, nb); scratch (N, 2, 4, nb); minv at REAL precision */
void CAT(ora_aux_pass, SFX)(int64_t n_cells, int nb, int nqv, int nqf, int maxf, const REAL *coeffs,
                            const REAL *qhat, const REAL *vol_w, const REAL *vol_basis, const REAL *vol_gx,
                            const REAL *vol_gy, const int8_t *cell_nfaces, const int32_t *cell_faces,
                            const int8_t *cell_fsign, const REAL *face_w, const REAL *fbL, const REAL *fbR,
                            const REAL *fnx, const REAL *fny, const REAL *minv, REAL *scratch, REAL *aux) {
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < n_cells; ++c) {
        REAL *sc = scratch + c * 8 * nb;
        for (int i = 0; i < 8 * nb; ++i) sc[i] = ZERO;
        const REAL *cc = coeffs + c * 4 * nb;
        for (int qp = 0; qp < nqv; ++qp) {
            REAL w = vol_w[c * nqv + qp];
            if (w == ZERO) continue;
            REAL qv[4] = {ZERO, ZERO, ZERO, ZERO};
            for (int k = 0; k < nb; ++k) {
                REAL b = vol_basis[(c * nqv + qp) * nb + k];
                for (int v = 0; v < 4; ++v) qv[v] += b * cc[v * nb + k];
            }
            for (int j = 0; j < nb; ++j) {
                REAL gx = w * vol_gx[(c * nqv + qp) * nb + j];
                REAL gy = w * vol_gy[(c * nqv + qp) * nb + j];
                for (int v = 0; v < 4; ++v) sc[(0 * 4 + v) * nb + j] -= qv[v] * gx;
                for (int v = 0; v < 4; ++v) sc[(1 * 4 + v) * nb + j] -= qv[v] * gy;
            }
        }
        for (int slot = 0; slot < cell_nfaces[c]; ++slot) {
            int64_t fid = cell_faces[c * maxf + slot];
            int sgn = cell_fsign[c * maxf + slot];
            const REAL *tb = sgn > 0 ? fbL : fbR;
            REAL s = (REAL)sgn;
            REAL nx = fnx[fid], ny = fny[fid];
            for (int q = 0; q < nqf; ++q) {
                REAL w = s * face_w[fid * nqf + q];
                const REAL *h = qhat + (fid * nqf + q) * 4;
                REAL wx = w * nx;
                REAL wy = w * ny;
                for (int j = 0; j < nb; ++j) {
                    REAL b = tb[(fid * nqf + q) * nb + j];
                    for (int v = 0; v < 4; ++v) sc[(0 * 4 + v) * nb + j] += h[v] * wx * b;
                    for (int v = 0; v < 4; ++v) sc[(1 * 4 + v) * nb + j] += h[v] * wy * b;
                }
            }
        }
        const REAL *mi = minv + c * nb * nb;
        for (int d = 0; d < 2; ++d)
            for (int v = 0; v < 4; ++v)
                for (int j = 0; j < nb; ++j) {
                    REAL acc = ZERO;
                    for (int k = 0; k < nb; ++k) acc += mi[j * nb + k] * sc[(d * 4 + v) * nb + k];
                    aux[((c * 2 + d) * 4 + v) * nb + j] = acc;
                }
    }
}

/* hodg/dg.py:240-351 with ivis = 1 (2D): Roe flux plus the central viscous
 * flux fvis and the trace average fqhat */
void CAT(ora_flux_pass_ns, SFX)(int64_t n_faces, int nqf, int nb, const REAL *coeffs, const REAL *aux, const REAL *fbL,
                                const REAL *fbR, const int32_t *face_cells, const int8_t *bc_code, const REAL *fnx,
                                const REAL *fny, const REAL *qinf, double gamma, double Rgas, double mu, double Pr,
                                REAL *finv, REAL *fvis, REAL *fqhat, uint8_t *errf) {
    const int d3 = 0;
    const REAL g = (REAL)gamma, R = (REAL)Rgas, m = (REAL)mu, pr = (REAL)Pr;
#pragma omp parallel for schedule(static)
    for (int64_t f = 0; f < n_faces; ++f) {
        int64_t iL = face_cells[2 * f], iR = face_cells[2 * f + 1];
        REAL n[2] = {fnx[f], fny[f]};
        for (int q = 0; q < nqf; ++q) {
            REAL qL[4] = {ZERO, ZERO, ZERO, ZERO}, qR[4] = {ZERO, ZERO, ZERO, ZERO};
            REAL zLx[4] = {ZERO, ZERO, ZERO, ZERO}, zLy[4] = {ZERO, ZERO, ZERO, ZERO};
            for (int k = 0; k < nb; ++k) {
                REAL b = fbL[(f * nqf + q) * nb + k];
                for (int v = 0; v < 4; ++v) qL[v] += b * coeffs[(iL * 4 + v) * nb + k];
            }
            for (int k = 0; k < nb; ++k) {
                REAL b = fbL[(f * nqf + q) * nb + k];
                for (int v = 0; v < 4; ++v) zLx[v] += b * aux[((iL * 2 + 0) * 4 + v) * nb + k];
                for (int v = 0; v < 4; ++v) zLy[v] += b * aux[((iL * 2 + 1) * 4 + v) * nb + k];
            }
            REAL zRx[4], zRy[4];
            for (int v = 0; v < 4; ++v) {
                zRx[v] = zLx[v];
                zRy[v] = zLy[v];
            }
            if (iR >= 0) {
                for (int k = 0; k < nb; ++k) {
                    REAL b = fbR[(f * nqf + q) * nb + k];
                    for (int v = 0; v < 4; ++v) qR[v] += b * coeffs[(iR * 4 + v) * nb + k];
                }
                for (int v = 0; v < 4; ++v) zRx[v] = zRy[v] = ZERO;
                for (int k = 0; k < nb; ++k) {
                    REAL b = fbR[(f * nqf + q) * nb + k];
                    for (int v = 0; v < 4; ++v) zRx[v] += b * aux[((iR * 2 + 0) * 4 + v) * nb + k];
                    for (int v = 0; v < 4; ++v) zRy[v] += b * aux[((iR * 2 + 1) * 4 + v) * nb + k];
                }
            } else {
                if (qL[0] <= ZERO) {
                    errf[f] = 1;
                    continue;
                }
                REAL u, v, w;
                REAL pL = CAT(prim_p, SFX)(qL[0], qL[1], qL[2], ZERO, qL[3], g, d3, &u, &v, &w);
                if (pL <= ZERO) {
                    errf[f] = 1;
                    continue;
                }
                CAT(bstate, SFX)(bc_code[f], qL, n, qinf, g, d3, qR);
            }
            REAL h[4];
            if (!CAT(roe, SFX)(qL, qR, n, g, d3, h)) {
                errf[f] = 1;
                continue;
            }
            for (int v = 0; v < 4; ++v) finv[(f * nqf + q) * 4 + v] = h[v];
            REAL hL[4], hR[4];
            CAT(viscn, SFX)(qL[0], qL[1], qL[2], qL[3], zLx, zLy, n[0], n[1], g, R, m, pr, hL);
            CAT(viscn, SFX)(qR[0], qR[1], qR[2], qR[3], zRx, zRy, n[0], n[1], g, R, m, pr, hR);
            for (int v = 0; v < 4; ++v) {
                fvis[(f * nqf + q) * 4 + v] = HALF * (hL[v] + hR[v]);
                fqhat[(f * nqf + q) * 4 + v] = HALF * (qL[v] + qR[v]);
            }
        }
    }
}

/* hodg/dg.py:353-460 with ivis = 1 (2D) */
void CAT(ora_rhs_pass_ns, SFX)(int64_t n_cells, int nb, int nqv, int nqf, int maxf, const REAL *coeffs,
                               const REAL *aux, const REAL *finv, const REAL *fvis, const REAL *vol_w,
                               const REAL *vol_basis, const REAL *vol_gx, const REAL *vol_gy,
                               const int8_t *cell_nfaces, const int32_t *cell_faces, const int8_t *cell_fsign,
                               const REAL *face_w, const REAL *fbL, const REAL *fbR, const double *minv64,
                               double gamma, double Rgas, double mu, double Pr, double *scratch, double *res,
                               uint8_t *errc) {
    const int d3 = 0;
    const REAL g = (REAL)gamma, R = (REAL)Rgas, m = (REAL)mu, pr = (REAL)Pr;
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < n_cells; ++c) {
        double *sc = scratch + c * 4 * nb;
        for (int i = 0; i < 4 * nb; ++i) sc[i] = 0.0;
        const REAL *cc = coeffs + c * 4 * nb;
        for (int qp = 0; qp < nqv; ++qp) {
            REAL w = vol_w[c * nqv + qp];
            if (w == ZERO) continue;
            REAL qv[4] = {ZERO, ZERO, ZERO, ZERO};
            for (int k = 0; k < nb; ++k) {
                REAL b = vol_basis[(c * nqv + qp) * nb + k];
                for (int v = 0; v < 4; ++v) qv[v] += b * cc[v * nb + k];
            }
            if (qv[0] <= ZERO) {
                errc[c] = 1;
                continue;
            }
            REAL u, v_, wz;
            REAL p = CAT(prim_p, SFX)(qv[0], qv[1], qv[2], ZERO, qv[3], g, d3, &u, &v_, &wz);
            if (p <= ZERO) {
                errc[c] = 1;
                continue;
            }
            REAL ex[4] = {qv[1], qv[1] * u + p, qv[1] * v_, (qv[3] + p) * u};
            REAL fy[4] = {qv[2], qv[2] * u, qv[2] * v_ + p, (qv[3] + p) * v_};
            REAL zx[4] = {ZERO, ZERO, ZERO, ZERO}, zy[4] = {ZERO, ZERO, ZERO, ZERO};
            for (int k = 0; k < nb; ++k) {
                REAL b = vol_basis[(c * nqv + qp) * nb + k];
                for (int vv = 0; vv < 4; ++vv) zx[vv] += b * aux[((c * 2 + 0) * 4 + vv) * nb + k];
                for (int vv = 0; vv < 4; ++vv) zy[vv] += b * aux[((c * 2 + 1) * 4 + vv) * nb + k];
            }
            REAL g8[8], s5[5];
            CAT(vel_temp_grads, SFX)(qv[0], qv[1], qv[2], qv[3], zx, zy, g, R, g8);
            CAT(stress_heat, SFX)(g8[2], g8[3], g8[4], g8[5], g8[6], g8[7], g, R, m, pr, s5);
            REAL uu = g8[0], vv2 = g8[1];
            ex[1] -= s5[0];
            ex[2] -= s5[1];
            ex[3] -= uu * s5[0] + vv2 * s5[1] - s5[3];
            fy[1] -= s5[1];
            fy[2] -= s5[2];
            fy[3] -= uu * s5[1] + vv2 * s5[2] - s5[4];
            for (int j = 0; j < nb; ++j) {
                REAL gx = w * vol_gx[(c * nqv + qp) * nb + j];
                REAL gy = w * vol_gy[(c * nqv + qp) * nb + j];
                for (int vv = 0; vv < 4; ++vv) sc[vv * nb + j] += ex[vv] * gx + fy[vv] * gy;
            }
        }
        for (int slot = 0; slot < cell_nfaces[c]; ++slot) {
            int64_t fid = cell_faces[c * maxf + slot];
            int sgn = cell_fsign[c * maxf + slot];
            const REAL *tb = sgn > 0 ? fbL : fbR;
            REAL s = (REAL)sgn;
            for (int q = 0; q < nqf; ++q) {
                REAL w = s * face_w[fid * nqf + q];
                REAL h[4];
                for (int vv = 0; vv < 4; ++vv) h[vv] = finv[(fid * nqf + q) * 4 + vv];
                for (int vv = 0; vv < 4; ++vv) h[vv] -= fvis[(fid * nqf + q) * 4 + vv];
                for (int j = 0; j < nb; ++j) {
                    REAL wb = w * tb[(fid * nqf + q) * nb + j];
                    for (int vv = 0; vv < 4; ++vv) sc[vv * nb + j] -= h[vv] * wb;
                }
            }
        }
        const double *mi = minv64 + c * nb * nb;
        for (int vv = 0; vv < 4; ++vv)
            for (int j = 0; j < nb; ++j) {
                double acc = 0.0;
                for (int k = 0; k < nb; ++k) acc += mi[j * nb + k] * sc[vv * nb + k];
                res[(c * 4 + vv) * nb + j] = acc;
            }
    }
}

/* Batched point evaluations of the interface flux and the boundary state
 * (the reference's Python API roe_flux / boundary_state,
 * hodg/physics.py:436-479).  q arrays are (n, nv), normals (n, dim). */
void CAT(ora_point_flux, SFX)(int dim, int64_t n, const REAL *qL, const REAL *qR, const REAL *nrm, double gamma,
                              int flux_kind, REAL *out, uint8_t *ok) {
    const int d3 = dim == 3;
    const int nv = d3 ? 5 : 4;
    for (int64_t i = 0; i < n; ++i) {
        ok[i] = (uint8_t)(flux_kind == 1 ? CAT(llf, SFX)(qL + i * nv, qR + i * nv, nrm + i * dim, (REAL)gamma, d3, out + i * nv)
                                         : CAT(roe, SFX)(qL + i * nv, qR + i * nv, nrm + i * dim, (REAL)gamma, d3, out + i * nv));
    }
}

void CAT(ora_point_bstate, SFX)(int dim, int64_t n, int kind, const REAL *q, const REAL *nrm, const REAL *qf,
                                double gamma, REAL *out) {
    const int d3 = dim == 3;
    const int nv = d3 ? 5 : 4;
    for (int64_t i = 0; i < n; ++i) CAT(bstate, SFX)(kind, q + i * nv, nrm + i * dim, qf, (REAL)gamma, d3, out + i * nv);
}

/* hodg/dg.py:240-351 (flux_pass, Euler branch), dimension-generic.
 * coeffs (N, nv, nb); fbL/fbR (F, nqf, nb); normal (dim, F) SoA;
 * finv (F, nqf, nv); errf (F,). */
void CAT(ora_flux_pass, SFX)(int dim, int64_t n_faces, int nqf, int nb, const REAL *coeffs, const REAL *fbL,
                             const REAL *fbR, const int32_t *face_cells, const int8_t *bc_code,
                             const REAL *normal, const REAL *qinf, double gamma, int flux_kind, REAL *finv,
                             uint8_t *errf) {
    const int d3 = dim == 3;
    const int nv = d3 ? 5 : 4;
    const REAL g = (REAL)gamma;
#pragma omp parallel for schedule(static)
    for (int64_t f = 0; f < n_faces; ++f) {
        int64_t iL = face_cells[2 * f], iR = face_cells[2 * f + 1];
        REAL n[3];
        for (int d = 0; d < dim; ++d) n[d] = normal[d * n_faces + f];
        for (int q = 0; q < nqf; ++q) {
            REAL qL[5] = {ZERO, ZERO, ZERO, ZERO, ZERO}, qR[5] = {ZERO, ZERO, ZERO, ZERO, ZERO};
            const REAL *bL = fbL + (f * nqf + q) * nb;
            for (int k = 0; k < nb; ++k) {
                REAL b = bL[k];
                for (int v = 0; v < nv; ++v) qL[v] += b * coeffs[(iL * nv + v) * nb + k];
            }
            if (iR >= 0) {
                const REAL *bR = fbR + (f * nqf + q) * nb;
                for (int k = 0; k < nb; ++k) {
                    REAL b = bR[k];
                    for (int v = 0; v < nv; ++v) qR[v] += b * coeffs[(iR * nv + v) * nb + k];
                }
            } else {
                if (qL[0] <= ZERO) {
                    errf[f] = 1;
                    continue;
                }
                REAL u, v, w;
                REAL pL = CAT(prim_p, SFX)(qL[0], qL[1], qL[2], d3 ? qL[3] : ZERO, QE(qL), g, d3, &u, &v, &w);
                if (pL <= ZERO) {
                    errf[f] = 1;
                    continue;
                }
                CAT(bstate, SFX)(bc_code[f], qL, n, qinf, g, d3, qR);
            }
            REAL h[5];
            int ok = flux_kind == 1 ? CAT(llf, SFX)(qL, qR, n, g, d3, h) : CAT(roe, SFX)(qL, qR, n, g, d3, h);
            if (!ok) {
                errf[f] = 1;
                continue;
            }
            for (int v = 0; v < nv; ++v) finv[(f * nqf + q) * nv + v] = h[v];
        }
    }
}

/* hodg/dg.py:353-460 (rhs_pass, Euler branch), dimension-generic.
 * vol_grad is (dim, N, nqv, nb); products in REAL, accumulation and the
 * mass-matrix solve in double. */
void CAT(ora_rhs_pass, SFX)(int dim, int64_t n_cells, int nb, int nqv, int nqf, int maxf, const REAL *coeffs,
                            const REAL *finv, const REAL *vol_w, const REAL *vol_basis, const REAL *vol_grad,
                            const int8_t *cell_nfaces, const int32_t *cell_faces, const int8_t *cell_fsign,
                            const REAL *face_w, const REAL *fbL, const REAL *fbR, const double *minv64,
                            double gamma, double *scratch, double *res, uint8_t *errc) {
    const int d3 = dim == 3;
    const int nv = d3 ? 5 : 4;
    const REAL g = (REAL)gamma;
    const int64_t gstride = n_cells * nqv * nb;
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < n_cells; ++c) {
        double *sc = scratch + c * nv * nb;
        for (int i = 0; i < nv * nb; ++i) sc[i] = 0.0;
        const REAL *cc = coeffs + c * nv * nb;
        for (int qp = 0; qp < nqv; ++qp) {
            REAL w = vol_w[c * nqv + qp];
            if (w == ZERO) continue;
            REAL qv[5] = {ZERO, ZERO, ZERO, ZERO, ZERO};
            const REAL *bb = vol_basis + (c * nqv + qp) * nb;
            for (int k = 0; k < nb; ++k) {
                REAL b = bb[k];
                for (int v = 0; v < nv; ++v) qv[v] += b * cc[v * nb + k];
            }
            if (qv[0] <= ZERO) {
                errc[c] = 1;
                continue;
            }
            REAL u, v_, wz;
            REAL p = CAT(prim_p, SFX)(qv[0], qv[1], qv[2], d3 ? qv[3] : ZERO, QE(qv), g, d3, &u, &v_, &wz);
            if (p <= ZERO) {
                errc[c] = 1;
                continue;
            }
            REAL E = QE(qv);
            /* physical fluxes in x, y, (z) */
            REAL fx[5], fy[5], fz[5];
            fx[0] = qv[1];
            fx[1] = qv[1] * u + p;
            fx[2] = qv[1] * v_;
            fy[0] = qv[2];
            fy[1] = qv[2] * u;
            fy[2] = qv[2] * v_ + p;
            if (d3) {
                fx[3] = qv[1] * wz;
                fy[3] = qv[2] * wz;
                fz[0] = qv[3];
                fz[1] = qv[3] * u;
                fz[2] = qv[3] * v_;
                fz[3] = qv[3] * wz + p;
                fz[4] = (E + p) * wz;
            }
            fx[nv - 1] = (E + p) * u;
            fy[nv - 1] = (E + p) * v_;
            const REAL *gxp = vol_grad + (c * nqv + qp) * nb;
            const REAL *gyp = gxp + gstride;
            const REAL *gzp = gyp + gstride;
            for (int j = 0; j < nb; ++j) {
                REAL gx = w * gxp[j];
                REAL gy = w * gyp[j];
                if (d3) {
                    REAL gz = w * gzp[j];
                    for (int v = 0; v < nv; ++v) sc[v * nb + j] += fx[v] * gx + fy[v] * gy + fz[v] * gz;
                } else {
                    for (int v = 0; v < nv; ++v) sc[v * nb + j] += fx[v] * gx + fy[v] * gy;
                }
            }
        }
        /* minus the surface integral of the stored interface fluxes */
        for (int slot = 0; slot < cell_nfaces[c]; ++slot) {
            int64_t fid = cell_faces[c * maxf + slot];
            int sgn = cell_fsign[c * maxf + slot];
            const REAL *tb = sgn > 0 ? fbL : fbR;
            REAL s = (REAL)sgn;
            for (int q = 0; q < nqf; ++q) {
                REAL w = s * face_w[fid * nqf + q];
                const REAL *h = finv + (fid * nqf + q) * nv;
                const REAL *bq = tb + (fid * nqf + q) * nb;
                for (int j = 0; j < nb; ++j) {
                    REAL wb = w * bq[j];
                    for (int v = 0; v < nv; ++v) sc[v * nb + j] -= h[v] * wb;
                }
            }
        }
        const double *mi = minv64 + c * nb * nb;
        for (int v = 0; v < nv; ++v)
            for (int j = 0; j < nb; ++j) {
                double acc = 0.0;
                for (int k = 0; k < nb; ++k) acc += mi[j * nb + k] * sc[v * nb + k];
                res[(c * nv + v) * nb + j] = acc;
            }
    }
}

/* hodg/timestepping.py:105-134 (_dt_pass): float64 arithmetic on the cell
 * mean; coeffs at state precision. */
void CAT(ora_dt_pass, SFX)(int dim, int64_t n_cells, int nb, const REAL *coeffs, const double *basis_mean,
                           const double *h, double gamma, double mu, double cfl, int order, double *out,
                           uint8_t *errc) {
    const int d3 = dim == 3;
    const int nv = d3 ? 5 : 4;
    const double fac = 2.0 * order + 1.0;
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < n_cells; ++c) {
        double m[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        for (int j = 0; j < nb; ++j) {
            double b = basis_mean[c * nb + j];
            for (int v = 0; v < nv; ++v) m[v] += b * (double)coeffs[(c * nv + v) * nb + j];
        }
        if (m[0] <= 0.0) {
            errc[c] = 1;
            out[c] = 0.0;
            continue;
        }
        double u = m[1] / m[0];
        double v = m[2] / m[0];
        double w = d3 ? m[3] / m[0] : 0.0;
        double E = m[nv - 1];
        double p = d3 ? (gamma - 1.0) * (E - 0.5 * m[0] * (u * u + v * v + w * w))
                      : (gamma - 1.0) * (E - 0.5 * m[0] * (u * u + v * v));
        if (p <= 0.0) {
            errc[c] = 1;
            out[c] = 0.0;
            continue;
        }
        double a = sqrt(gamma * p / m[0]);
        double speed = (d3 ? sqrt(u * u + v * v + w * w) : sqrt(u * u + v * v)) + a +
                       2.0 * mu * fac / (m[0] * h[c]);
        out[c] = cfl * h[c] / (fac * speed);
    }
}

/* hodg/timestepping.py:165-171 (_axpy_state): out = u + dt r, computed in
 * double, stored at state precision. */
void CAT(ora_axpy, SFX)(int64_t n_cells, int per_cell, const REAL *u, const double *r, const double *dtc,
                        REAL *out) {
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < n_cells; ++c) {
        double dt = dtc[c];
        for (int i = 0; i < per_cell; ++i) {
            int64_t k = c * per_cell + i;
            out[k] = (REAL)((double)u[k] + dt * r[k]);
        }
    }
}

/* hodg/timestepping.py:174-180 (_combine_state): out = (u + u1 + dt r1)/2;
 * u + u1 is evaluated at state precision (numba keeps float32+float32 in
 * float32) before promotion. */
void CAT(ora_combine, SFX)(int64_t n_cells, int per_cell, const REAL *u, const REAL *u1, const double *r1,
                           const double *dtc, REAL *out) {
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < n_cells; ++c) {
        double dt = dtc[c];
        for (int i = 0; i < per_cell; ++i) {
            int64_t k = c * per_cell + i;
            REAL s = u[k] + u1[k];
            out[k] = (REAL)(0.5 * ((double)s + dt * r1[k]));
        }
    }
}

/* SSP-RK3 stage combination (not in the reference, which is RK2 only):
 * out = a u + b (us + dt r), double arithmetic, stored at state precision. */
void CAT(ora_rk_combo, SFX)(int64_t n_cells, int per_cell, double a, double b, const REAL *u, const REAL *us,
                            const double *r, const double *dtc, REAL *out) {
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < n_cells; ++c) {
        double dt = dtc[c];
        for (int i = 0; i < per_cell; ++i) {
            int64_t k = c * per_cell + i;
            out[k] = (REAL)(a * (double)u[k] + b * ((double)us[k] + dt * r[k]));
        }
    }
}

#undef ONE
#undef ZERO
#undef HALF
#undef TWO
#undef QUARTER
#undef EFIX
#undef QE
