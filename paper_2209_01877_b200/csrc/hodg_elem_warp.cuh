// Warp-group element kernel (P1, P2): hodg/dg.py:353-460 (rhs_pass, Euler
// branch) fused with the RK stage update (hodg/timestepping.py:165-180) and
// the next step's CFL dt (hodg/timestepping.py:105-134).  Included inside
// namespace hodg::ord<ORDER> by hodg_kernels.cuh.
//
// Each warp owns groups of G = 6 elements; lane (e, v) = (lane / 5, lane % 5)
// holds element e's variable v (lanes 30, 31 idle).  The warps of a CTA
// share nothing, so there is no CTA barrier anywhere: only __syncwarp.
// Persistent: warp w loops over groups w, w + W, ...  The next group's state
// rows, geometry and face ids are TMA bulk copies issued as soon as the
// current group's coefficients are in registers; the current group's face
// flux records are cp.async 16-byte chunks spread over the element's five
// lanes (a handful of instructions per lane, no per-record copy-issue loop),
// in flight during the volume integral.
//
// Volume integral through the monomial-derivative identity
//   VD[q][i][d] = w_q dm_i/deta_d (eta_q) = alpha_{i,d} w_q m_{i - e_d}(eta_q):
// the lane accumulates the moments MOM[j][k] = sum_q w_q m_j(eta_q) F_vk(q)
// of its variable's physical flux against the NBL monomials of degree
// < ORDER, and applies J^-1 once at the end:
//   sum_q sum_d VD[q][i][d] (J^-1 F)_d = sum_d alpha_{i,d} sum_k Jinv[d][k] MOM[i - e_d][k].
// At each quadrature point the five lanes of an element exchange their
// traces through shared memory and each recovers the primitive state itself
// (no second exchange): F_v,d = U_v vel_d + p (delta_{v,d+1} + delta_{v,4} vel_d).

#ifndef HODG_WPC
#define HODG_WPC 2  // warps per CTA
#endif
#ifndef HODG_WMINB
#define HODG_WMINB 9  // CTAs per SM the register budget is set for
#endif
constexpr int WPC = HODG_WPC;

template <typename T, bool ES>
struct WarpSmem {
    static constexpr size_t bar = 0;                              // in[2] (state + geometry + face ids), rec
    static constexpr size_t st = 32;                              // G x RS doubles (one buffer)
    static constexpr size_t geo = st + align16(size_t(G) * RS * 8);  // [2][16][G] doubles
    static constexpr size_t fid = geo + size_t(2) * 16 * G * 8;   // [2][4][G] int32
    static constexpr size_t rec = align16(fid + size_t(2) * 4 * G * 4);
    static constexpr size_t rec_bytes =
        ES ? align16(size_t(G) * EREC * sizeof(T)) : size_t(4) * G * hstride<T>() * sizeof(T);
    static constexpr size_t xs = align16(rec + rec_bytes);        // 2 x 32 exchange slots
    static constexpr size_t total = align16(xs + 2 * 32 * 8);
};

template <typename T, bool ES>
__host__ __device__ constexpr size_t warp_smem_bytes() {
    return size_t(WPC) * WarpSmem<T, ES>::total;
}

// 16-byte aligned global row segment -> registers
template <int N>
__device__ __forceinline__ void ldg_row(const double* __restrict__ src, double (&dst)[N]) {
#pragma unroll
    for (int k = 0; k + 1 < N; k += 2) {
        const double2 p = __ldg(reinterpret_cast<const double2*>(src + k));
        dst[k] = p.x;
        dst[k + 1] = p.y;
    }
    if constexpr (N % 2 == 1) dst[N - 1] = __ldg(src + N - 1);
}

template <typename T, bool ES>
__global__ void __launch_bounds__(WPC * 32, HODG_WMINB)
    elem_warp_kernel(const hodg_mesh_desc m, const T* __restrict__ hbuf, const hodg_stage_args a,
                     uint32_t* __restrict__ err) {
    using L = WarpSmem<T, ES>;
    constexpr int HS = hstride<T>();
    constexpr int NC16 = int(HS * sizeof(T) / 16);  // 16-byte chunks per face record
    extern __shared__ __align__(16) unsigned char smem_all[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    unsigned char* smem = smem_all + size_t(warp) * L::total;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::bar);
    double* ST = reinterpret_cast<double*>(smem + L::st);
    double* GEO = reinterpret_cast<double*>(smem + L::geo);
    int32_t* FID = reinterpret_cast<int32_t*>(smem + L::fid);
    T* REC = reinterpret_cast<T*>(smem + L::rec);
    double* XS = reinterpret_cast<double*>(smem + L::xs);

    const int e = lane / 5;
    const int v = lane - 5 * e;
    const int ex = e < G ? e : G - 1;  // idle lanes 30, 31 read a live element's slots
    const int64_t ngroups = (m.n_elems + G - 1) / G;
    const int64_t wstride = int64_t(gridDim.x) * WPC;
    int64_t g = int64_t(blockIdx.x) * WPC + warp;
    if (a.dt_reset && blockIdx.x == 0 && threadIdx.x == 0) *a.dt_reset = 0x7FF0000000000000ull;

    auto issue_inputs = [&](int64_t gg, int buf) {  // lane 0
        const int ne = int(min(int64_t(G), m.n_elems - gg * G));
        const uint32_t bs = uint32_t(ne) * RS * 8;
        mbar_arrive_expect_tx(bar + buf, bs + 16 * G * 8 + 4 * G * 4);
        bulk_g2s(ST, a.us + gg * G * RS, bs, bar + buf);
        bulk_g2s(GEO + buf * 16 * G, m.egeo + gg * 16 * G, 16 * G * 8, bar + buf);
        bulk_g2s(FID + buf * 4 * G, m.efaces + gg * 4 * G, 4 * G * 4, bar + buf);
    };
    if (lane == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        mbar_init(bar + 2, 1);
        mbar_fence_init();
    }
    __syncwarp();
    if (lane == 0 && g < ngroups) issue_inputs(g, 0);
    // programmatic dependent launch: the state was produced two launches
    // back; the face records and the in-place output need the previous
    // launch complete
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");

    const bool need_u0 = a.combine == 1 || (a.combine == 0 && a.a != 0.0);
    const T gam = T(m.gamma);
    const T gm1 = gam - T(1);
    // flux selectors of this lane's variable
    const T kd0 = v == 1 ? T(1) : T(0), kd1 = v == 2 ? T(1) : T(0), kd2 = v == 3 ? T(1) : T(0);
    const T k4 = v == 4 ? T(1) : T(0);
    unsigned long long dtmin = 0x7FF0000000000000ull;

    for (int it = 0; g < ngroups; g += wstride, ++it) {
        const int buf = it & 1;
        const int64_t e0 = g * G;
        const int ne = int(min(int64_t(G), m.n_elems - e0));
        const bool live = e < ne;
        const int64_t gid = e0 + e;
        const double* gb = GEO + buf * 16 * G;
        mbar_wait(bar + buf, (it >> 1) & 1);

        // this group's face flux records, in flight during the volume integral
        if constexpr (ES) {
            if (lane == 0) {
                const uint32_t hb = uint32_t(align16(size_t(ne) * EREC * sizeof(T)));
                mbar_arrive_expect_tx(bar + 2, hb);
                bulk_g2s(REC, hbuf + e0 * EREC, hb, bar + 2);
            }
        } else {
            if (live) {
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    const int64_t f = FID[buf * 4 * G + s * G + e];
                    const char* src = reinterpret_cast<const char*>(hbuf + f * HS);
                    char* dst = reinterpret_cast<char*>(REC + (s * G + e) * HS);
#pragma unroll
                    for (int ch = v; ch < NC16; ch += 5) cp_async16(dst + 16 * ch, src + 16 * ch);
                }
            }
            cp_async_commit();
        }

        // coefficients of (e, v), then the state buffer is free for the next group
        double c[NB];
        ld_row(ST + ex * RS + v * NB, c);
        __syncwarp();
        if (lane == 0 && g + wstride < ngroups) {
            fence_proxy_async();
            issue_inputs(g + wstride, buf ^ 1);
        }

        // ---- volume integral: moments of this variable's flux --------------
        T cf[NB];
#pragma unroll
        for (int i = 0; i < NB; ++i) cf[i] = T(c[i]);
        T mom[NBL][3];
#pragma unroll
        for (int j = 0; j < NBL; ++j) mom[j][0] = mom[j][1] = mom[j][2] = T(0);
        bool bad = false;
        sfor<NQV>([&](auto q) {
            // trace of variable v (two partial sums: shorter dependency chain)
            T u0 = T(0), u1 = T(0);
            sfor<NB>([&](auto i) {
                if constexpr (i % 2 == 0) u0 += TAB(VB, T, q * NB + i) * cf[i];
                else u1 += TAB(VB, T, q * NB + i) * cf[i];
            });
            const T u = u0 + u1;
            T* xq = reinterpret_cast<T*>(XS + (q & 1) * 32);
            xq[lane] = u;
            __syncwarp();
            T U[5];
#pragma unroll
            for (int k = 0; k < 5; ++k) U[k] = xq[ex * 5 + k];
            const T ri = rcp_nr(U[0]);
            const T vx = U[1] * ri, vy = U[2] * ri, vz = U[3] * ri;
            const T pr = gm1 * (U[4] - T(0.5) * (U[1] * vx + U[2] * vy + U[3] * vz));
            if ((U[0] > T(0)) && (pr > T(0))) {
                const T F0 = u * vx + pr * (kd0 + k4 * vx);
                const T F1 = u * vy + pr * (kd1 + k4 * vy);
                const T F2 = u * vz + pr * (kd2 + k4 * vz);
                sfor<NBL>([&](auto j) {
                    const T wm = TAB(WV, T, q * NB + j);
                    mom[j][0] += wm * F0;
                    mom[j][1] += wm * F1;
                    mom[j][2] += wm * F2;
                });
            } else {
                bad = true;  // zero flux at this point, as the reference's flagged cell
            }
        });
        if (bad && live && v == 0) flag(err, 1, uint32_t(gid));
        // J^-1 once: mj[j][d] = sum_k Jinv[d][k] mom[j][k]; then the derivative identity
        T acc[NB];
        {
            T ji[9];
#pragma unroll
            for (int k = 0; k < 9; ++k) ji[k] = T(gb[k * G + ex]);
            T mj[NBL][3];
#pragma unroll
            for (int j = 0; j < NBL; ++j)
#pragma unroll
                for (int d = 0; d < 3; ++d)
                    mj[j][d] = ji[3 * d] * mom[j][0] + ji[3 * d + 1] * mom[j][1] + ji[3 * d + 2] * mom[j][2];
            sfor<NB>([&](auto i) {
                T s = T(0);
                sfor<3>([&](auto d) {
                    constexpr int al = expt(i, d);
                    if constexpr (al > 0) {
                        constexpr int lo = mono_index(expt(i, 0) - (d == 0), expt(i, 1) - (d == 1), expt(i, 2) - (d == 2));
                        s += T(al) * mj[lo][d];
                    }
                });
                acc[i] = s;
            });
        }

        // RK base state, in flight during the gather
        double u0r[NB];
        if (need_u0 && live) ldg_row(a.u0 + gid * RS + v * NB, u0r);

        // ---- face gather -----------------------------------------------------
        if constexpr (ES) {
            mbar_wait(bar + 2, it & 1);
        } else {
            cp_async_wait_all();
            __syncwarp();
        }
        double accd[NB];
#pragma unroll
        for (int i = 0; i < NB; ++i) accd[i] = double(acc[i]);
        sfor<4>([&](auto s) {
            const T* hrec = ES ? REC + ex * EREC + s * HSE + v * NQF : REC + (s * G + ex) * HS + v * NQF;
            T hq[NQF];
#pragma unroll
            for (int q = 0; q < NQF; ++q) hq[q] = hrec[q];
            T fa[NB];
            face_moments<T, s, 0, NB>(hq, fa);
            const double fc = gb[(9 + s) * G + ex];
#pragma unroll
            for (int i = 0; i < NB; ++i) accd[i] -= fc * double(fa[i]);
        });

        // ---- mass solve (FP64, constant reference MINV) ------------------------
        double r[NB];
        sfor<NB>([&](auto j) {
            double z = 0.0;
            sfor<NB>([&](auto k) { z += MINV_T[j * NB + k] * accd[k]; });
            r[j] = z;
        });
        if (a.res && live) {
#pragma unroll
            for (int j = 0; j + 1 < NB; j += 2)
                *reinterpret_cast<double2*>(a.res + gid * RS + v * NB + j) = make_double2(r[j], r[j + 1]);
        }
        // residual-norm partial of this group: sum over its elements in order
        if (a.norm_partial) {
            const double term = live ? gb[14 * G + ex] * r[0] * r[0] : 0.0;
            XS[lane] = term;
            __syncwarp();
            if (lane < 5) {
                double sum = 0.0;
                for (int ee = 0; ee < ne; ++ee) sum += XS[ee * 5 + lane];
                a.norm_partial[g * 5 + lane] = sum;
            }
        }
        // ---- RK combination, new state, CFL dt of its cell mean ----------------
        if (a.combine >= 0) {
            const double dt = a.dt_is_vector ? (live ? a.dt[gid] : 0.0) : a.dt[0];
            double o[NB];
            double mean = 0.0;
            sfor<NB>([&](auto j) {
                double oj;
                if (a.combine == 1) {
                    oj = 0.5 * ((u0r[j] + c[j]) + dt * r[j]);
                } else {
                    oj = a.b * (c[j] + dt * r[j]);
                    if (a.a != 0.0) oj = a.a * u0r[j] + oj;
                }
                o[j] = oj;
                mean += MEAN_T[j] * oj;
            });
            if (live) {
#pragma unroll
                for (int j = 0; j + 1 < NB; j += 2)
                    *reinterpret_cast<double2*>(a.out + gid * RS + v * NB + j) = make_double2(o[j], o[j + 1]);
                if constexpr (sizeof(T) == 4) {
                    if (a.out32) {  // mixed: the FP32 shadow the next face kernel reads
#pragma unroll
                        for (int j = 0; j + 1 < NB; j += 2)
                            *reinterpret_cast<float2*>(a.out32 + gid * RSF + v * NB + j) =
                                make_float2(float(o[j]), float(o[j + 1]));
                    }
                }
            }
            if (a.dt_next || a.dt_vec_out) {
                // the five variable means of element e, at its v == 0 lane
                double mm[5];
                mm[0] = mean;
#pragma unroll
                for (int k = 1; k < 5; ++k) mm[k] = __shfl_sync(0xffffffffu, mean, (ex * 5 + k) & 31);
                if (live && v == 0) {
                    double dte = 0.0;
                    bool okdt = false;
                    const double m0 = mm[0];
                    if (!(m0 > 0.0)) {
                        flag(err, 2, uint32_t(gid));
                    } else {
                        const double ri = 1.0 / m0;
                        const double uu = mm[1] * ri, vv = mm[2] * ri, ww = mm[3] * ri;
                        const double p = (m.gamma - 1.0) * (mm[4] - 0.5 * m0 * (uu * uu + vv * vv + ww * ww));
                        if (!(p > 0.0)) {
                            flag(err, 2, uint32_t(gid));
                        } else {
                            const double speed = sqrt(uu * uu + vv * vv + ww * ww) + sqrt(m.gamma * p * ri);
                            dte = a.cfl * gb[13 * G + ex] / ((2.0 * ORDER + 1.0) * speed);
                            okdt = true;
                        }
                    }
                    if (a.dt_vec_out) a.dt_vec_out[gid] = dte;
                    if (okdt) {
                        const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(dte));
                        dtmin = bits < dtmin ? bits : dtmin;
                    }
                }
            }
        }
        __syncwarp();  // exchange slots and records consumed before the next group
    }
    if (a.combine >= 0 && a.dt_next) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long other = __shfl_xor_sync(0xffffffffu, dtmin, o);
            dtmin = other < dtmin ? other : dtmin;
        }
        if (lane == 0 && dtmin != 0x7FF0000000000000ull) atomicMin(a.dt_next, dtmin);
    }
}
