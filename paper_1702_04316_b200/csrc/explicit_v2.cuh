// explicit_v2.cuh -- production explicit-stage kernel (included by hevi.cu
// inside its anonymous namespace).
//
// One CTA per horizontal tile of TX x TY element columns sweeps the element
// layers bottom-up.  Per layer:
//   1. TMA (cp.async.bulk.tensor, 4D box x,y,1 level,5 fields) writes each
//      new level of the tile plus its low-side halo straight into its slot of
//      a ring of 2N+1 level slots (the top level of a layer is the bottom of
//      the next).  Two layers are resident: while layer ez computes, the N
//      levels of layer ez+1 are in flight, issued at the end of layer ez-1
//      (two mbarriers, one per layer parity), so a load has a whole layer of
//      compute to land and nothing is copied between shared buffers;
//   2. P' of the layer's new levels is formed in place (6th plane of the
//      slot).  P' = EOS(rho, theta) - P0f
//      (euler.py:454-457) is evaluated as Pb (1+delta)^gamma - P0f with
//      delta = (rho theta - rho0 theta0)/(rho0 theta0) by its binomial series
//      (15 terms, |delta| <= 1/8; exact pow beyond): the same function,
//      ~20 FMAs instead of a ~240-instruction pow, and no cancellation;
//   3. per-layer partial sums that more than one point needs are formed once:
//      row N of the left element at element x-faces, row N of this layer at
//      its top face (the carry into the next layer's bottom face);
//   4. one thread per owned lattice point: 19 derivative lines with the
//      thread's D rows held in registers for the whole sweep, R(q) and
//      L_V(q) pointwise, no-flux projection, fused ARK2 stage epilogue.
#pragma once

// The pointwise stage inputs A / F of the layer's owned points arrive by TMA
// (4D box OX x OYM x N x 5) issued at the start of the layer and are read from
// shared memory in the epilogue (no registers held through the derivative
// phase, no exposed global latency); even N only (x origin must be even).
// Measured at config 5: M_S2 (stage 1) 1.659 -> 1.584 ms; M_S3 (stage 2, F
// only) 1.402 -> 1.475 ms, so M_S3 keeps its early register loads.
#ifndef HEVI_X_AFTMA_MASK
#define HEVI_X_AFTMA_MASK (1 << M_S2)
#endif
// Per mode (bit MODE): form the x-face partials of the 5 state fields in the
// P' phase and let the face points take their own P' face line, which drops
// one barrier per layer.  Measured at config 5: stage 0 (M_S1) 1.581 -> 1.548
// ms, stage 2 (M_S3) 1.443 -> 1.402 ms, stage 1 (M_S2, with its A/F boxes
// staged by TMA) 1.584 -> 1.537 ms (before the A/F staging it was slower).
#ifndef HEVI_X_XF6
#define HEVI_X_XF6 1   // with the P' plane staged, its face partials join the merged face phase (-1%)
#endif
#ifndef HEVI_X_MERGE_MASK
#define HEVI_X_MERGE_MASK 63
#endif

#ifndef HEVI_X_TREE
#define HEVI_X_TREE 0   // 1: line sums as two interleaved chains (depth ~N/2 + 1)
#endif
// sum_m D[m] s[m*STR], m = 0..NN: one chain (reference order) or two
// interleaved chains joined at the end (shorter dependency path)
template <int NN, int STR>
__device__ __forceinline__ double line_sum(const double* D, const double* s) {
    if (HEVI_X_TREE && NN >= 3) {
        double a = D[0] * s[0], b = D[1] * s[STR];
#pragma unroll
        for (int m = 2; m <= NN; m += 2) {
            a = fma(D[m], s[m * STR], a);
            if (m + 1 <= NN) b = fma(D[m + 1], s[(m + 1) * STR], b);
        }
        return a + b;
    }
    double d = 0.0;
#pragma unroll
    for (int m = 0; m <= NN; ++m) d = fma(D[m], s[m * STR], d);
    return d;
}

__device__ __forceinline__ void pf_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

template <int N, int NY>
struct Tile2;   // TX, TY, MINB (defined with the dispatch in hevi.cu)

template <int N, int NY, int TX, int TY>
struct E2 {
    static constexpr int OX = TX * N;                         // main x points per tile
    static constexpr int OYM = TY * NY + (NY == 1 ? 1 : 0);   // main y rows (slab: both)
    static constexpr int LX = OX + N + 1;                     // loaded x extent (low halo N)
    // TMA box x: 16-byte multiple and one spare column, because the box
    // x-origin is floored to an even index (an odd, negative origin is an
    // illegal TMA request on sm_100a; tools/tma_probe.cu)
    static constexpr int LXT = (LX + 2) / 2 * 2;
    static constexpr int LY = TY * NY + NY + 1;
    static constexpr int NL = N + 1;                          // levels per layer
    static constexpr int RING = 2 * N + 1;                    // level slots (two layers)
    static constexpr int PL = LY * LXT;                       // one field plane of a level
    // P' plane of a slot at a 128-byte aligned offset (it can arrive by its own TMA)
    static constexpr int PPO = (5 * PL + 15) / 16 * 16;
    static constexpr int SS = (PPO + PL + 15) / 16 * 16;      // slot stride (128-byte aligned)
    __host__ __device__ static constexpr int foff(int f) { return f < 5 ? f * PL : PPO; }
#ifdef HEVI_X_K
    static constexpr int K = HEVI_X_K;
#else
    static constexpr int K = (N % 2 == 0) ? 2 : 1;             // vertical points per thread
#endif
    static constexpr int NT = OX * OYM * (N / K);             // main threads
    static constexpr int BLK = (NT + 31) / 32 * 32;
    static constexpr int CXW = OX + 1, CYW = TY * NY + 1 + (NY == 1 ? 1 : 0);
    static constexpr int S_N = RING * SS;                     // ring: rho', u, v, w, theta', P'
    static constexpr int CAR_N = 2 * 7 * CYW * CXW;           // double-buffered carry
    static constexpr int XF_N = 6 * TX * OYM * N;             // x-face partials
    static constexpr int DN = (N + 1) * (N + 1), DNY = (NY + 1) * (NY + 1);
    static constexpr int AFB = OX * OYM * N * 5;                 // one A or F layer box
    static constexpr int AF_N = (HEVI_X_AFTMA_MASK && N % 2 == 0) ? 2 * AFB : 0;
    static constexpr uint32_t AF_BYTES = (uint32_t)(sizeof(double) * AFB);
    // shared bytes of a mode (the A/F boxes only where that mode stages them)
    __host__ __device__ static constexpr int af_of(int mode) { return ((HEVI_X_AFTMA_MASK >> mode) & 1) ? AF_N : 0; }
    static constexpr size_t fixed_bytes(int mode = -1) {
        return sizeof(double) * (size_t)(S_N + (mode < 0 ? AF_N : af_of(mode)) + CAR_N + XF_N + DN +
                                         DNY + 3) + 128;
    }
    static constexpr int NTAB = 12;                           // level tables in smem
    static constexpr uint32_t LVL_BYTES = (uint32_t)(sizeof(double) * 5 * PL);   // one level TMA
    static constexpr uint32_t PP_BYTES = (uint32_t)(sizeof(double) * PL);        // its P' plane
};

// smem level tables
enum { T_RHO0 = 0, T_TH0, T_E0, T_C0, T_IRT0, T_G0, T_H0, T_DRHO0, T_DTH0, T_CZ, T_P0F, T_IRHO0 };

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
                 "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
        "l"(map), "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

// shorter series for |delta| <= 2^-10 (the usual case: acoustic perturbations)
#ifndef HEVI_PP_SHORT
#define HEVI_PP_SHORT 1
#endif

// the rare |delta| > 1/8 branch of P', out of line: one copy per kernel
// instead of one per inlined call site (the column kernels' code size and
// register budget)
__device__ __noinline__ double pprime_pow(double rho, double theta, double P0f, double P0, double R,
                                          double gamma) {
    return P0 * pow(rho * R * theta / P0, gamma) - P0f;
}

// P' at one point; rho0/theta0/Pb/c0/irt0 of its level
__device__ __forceinline__ double pprime(double r, double th, double rho0, double th0, double Pb,
                                         double c0, double irt0, double P0f, const double* bc,
                                         const Phys& ph) {
    const double delta = (r * th0 + th * (rho0 + r)) * irt0;
    if (HEVI_PP_SHORT && fabs(delta) <= 0x1p-10) {
        // |delta| <= 2^-10: the terms beyond delta^6 are below 1e-20 relative
        double s = bc[5];
#pragma unroll
        for (int k = 4; k >= 0; --k) s = fma(s, delta, bc[k]);
        return fma(Pb, s * delta, c0);
    }
    if (fabs(delta) <= 0.125) {
        double s = bc[14];
#pragma unroll
        for (int k = 13; k >= 0; --k) s = fma(s, delta, bc[k]);
        return fma(Pb, s * delta, c0);
    }
    return pprime_pow(rho0 + r, th0 + th, P0f, ph.P0, ph.R, ph.gamma);
}

template <int N, int NY, int K>
struct DRows {
    double x[N + 1], y[NY + 1], z[K][N + 1];   // the points' own rows; face rows (row N) from smem
};

// per-axis geometry of one point inside the tile
struct PAx {
    int l, s0, row;
    bool face;
};

__device__ __forceinline__ PAx pax(int gi, int l, int N, int ne) {
    PAx r;
    r.l = l;
    if (gi == ne * N) {
        r.row = N;
        r.s0 = l - N;
        r.face = false;
    } else {
        r.row = gi % N;
        r.s0 = l - r.row;
        r.face = (r.row == 0) && (gi > 0);
    }
    return r;
}

// K vertically adjacent points (levels oz0 .. oz0+K-1 of one column) per
// thread: x/y rows and set-up are shared, every z-line is loaded once for
// all K points, and the K derivative chains are independent (ILP).
template <int N, int NY, int TX, int TY, int MODE, bool MAIN, int K>
__device__ __forceinline__ void e2_pts(const EArgs& a, const double* __restrict__ S,
                                       const double* __restrict__ CARp, double* __restrict__ CARw,
                                       const double* __restrict__ XF, const double* __restrict__ LT,
                                       const DRows<N, NY, K>& D, const double* __restrict__ sDx,
                                       const double* __restrict__ sDy, const PAx& ax, const PAx& ay,
                                       int oz0, int ox, int oy, int gx, int gy, int ez, double cx,
                                       double cy, int Z, const double* __restrict__ sAF = nullptr,
                                       uint64_t* mbaf = nullptr, bool xf5 = false) {
    using T = E2<N, NY, TX, TY>;
    constexpr int PL = T::PL, LXT = T::LXT, RING = T::RING, SS = T::SS;
    constexpr bool NEED_L = (MODE == M_L || MODE == M_S1 || MODE == M_S2);
    constexpr bool NEED_R = (MODE != M_L);
    const Geo& g = a.g;
    const long long fs = g.fs;
    const int base = ez * N;
    (void)mbaf;
    long long o[K];
    int sl[K], gzk[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        gzk[k] = base + oz0 + k;
        o[k] = loff(g, gx, gy, gzk[k]);
        sl[k] = (base + oz0 + k) % RING;
    }
    // stage inputs read pointwise: issue early, consume in the epilogue
    // (MAIN points with a staged A/F box read them from shared memory instead)
    double Ain[K][5], Fin[K][5];
    const bool af_smem = MAIN && T::AF_N > 0 && sAF != nullptr && ((HEVI_X_AFTMA_MASK >> MODE) & 1);
#pragma unroll
    for (int k = 0; k < K && !af_smem; ++k) {
        if (MODE == M_S2 || (MODE == M_RK && a.A != nullptr)) {
#pragma unroll
            for (int f = 0; f < 5; ++f) Ain[k][f] = a.A[o[k] + f * fs];
        }
        if (MODE == M_S2 || MODE == M_S3) {
#pragma unroll
            for (int f = 0; f < 5; ++f) Fin[k][f] = a.F[o[k] + f * fs];
        }
    }
    int zs[N + 1];
#pragma unroll
    for (int m = 0; m <= N; ++m) zs[m] = ((base + m) % RING) * SS;
    const int cidx = oy * T::CXW + ox;
    const bool more = ez + 1 < g.nez;
    const bool do_carry = (oz0 == 0) && more;
    const bool zface = (oz0 == 0) && (ez > 0);
    const double* Sxy = S + ay.l * LXT + ax.l;   // column base (plus slot*SS + f*PL)

    double r[K], u[K], v[K], w[K], th[K], rho[K], rinv[K], cz[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const double* pp = Sxy + sl[k] * SS;
        r[k] = pp[0 * PL];
        u[k] = pp[1 * PL];
        v[k] = pp[2 * PL];
        w[k] = pp[3 * PL];
        th[k] = pp[4 * PL];
        rho[k] = LT[gzk[k] * T::NTAB + T_RHO0] + r[k];
        rinv[k] = 1.0 / rho[k];
        cz[k] = LT[gzk[k] * T::NTAB + T_CZ];
    }
    // d/dx, d/dy, d/dz of field f at the K points (DSS-averaged, folded)
    // per-layer line base addresses: every line load below is base + a
    // compile-time offset (field * SF + m * stride)
    constexpr int SF = PL;
    const double* bx_[K];
    const double* bxl_[K];
    const double* by_[K];
    const double* byl_[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        bx_[k] = S + sl[k] * SS + ay.l * LXT + ax.s0;
        bxl_[k] = S + sl[k] * SS + ay.l * LXT + ax.l - N;
        by_[k] = S + sl[k] * SS + ay.s0 * LXT + ax.l;
        byl_[k] = S + sl[k] * SS + (ay.l - NY) * LXT + ax.l;
    }
    const double* bz_[N + 1];
#pragma unroll
    for (int m = 0; m <= N; ++m) bz_[m] = S + zs[m] + ay.l * LXT + ax.l;
    const double* xfp = XF + ((TX == 0 ? 0 : ox / N) * T::OYM + oy) * N + oz0;
    const double* carp = CARp + cidx;
    double* carw = CARw + cidx;
    // d/dx, d/dy, d/dz of field f at the K points (DSS-averaged, folded)
    auto grad = [&](int f, bool want_xy, double (&gxv)[K], double (&gyv)[K], double (&gzv)[K]) {
        if (want_xy) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const double* sx = bx_[k] + T::foff(f);
                double d = line_sum<N, 1>(D.x, sx);
                if (MAIN && !(((HEVI_X_MERGE_MASK >> MODE) & 1) && f == 5 && !xf5)) {
                    // branch-free: the XF slot is in bounds for every main point
                    const double xf = xfp[f * (TX * T::OYM * N) + k];
                    d += ax.face ? xf : 0.0;
                } else if (ax.face) {
                    {
                        const double* sxl = bxl_[k] + T::foff(f);
                        double e = 0.0;
#pragma unroll
                        for (int m = 0; m <= N; ++m) e = fma(sDx[N * (N + 1) + m], sxl[m], e);
                        d += e;
                    }
                }
                gxv[k] = cx * d;
                const double* sy = by_[k] + T::foff(f);
                double e = line_sum<NY, LXT>(D.y, sy);
                if (ay.face) {
                    const double* syl = byl_[k] + T::foff(f);
                    double h = 0.0;
#pragma unroll
                    for (int m = 0; m <= NY; ++m) h = fma(sDy[NY * (NY + 1) + m], syl[m * LXT], h);
                    e += h;
                }
                gyv[k] = cy * e;
            }
        }
        double val[N + 1];
        if (f == 6) {
            // linearised pressure G0 rho' + H0 theta' (euler.py:188-194) on the z-line
#pragma unroll
            for (int m = 0; m <= N; ++m)
                val[m] = LT[(base + m) * T::NTAB + T_G0] * bz_[m][0] + LT[(base + m) * T::NTAB + T_H0] * bz_[m][4 * SF];
        } else {
#pragma unroll
            for (int m = 0; m <= N; ++m) val[m] = bz_[m][T::foff(f)];
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double d = line_sum<N, 1>(D.z[k], val);
            if (k == 0) {
                const double cr = carp[f * (T::CYW * T::CXW)];
                d += zface ? cr : 0.0;
            }
            gzv[k] = cz[k] * d;
        }
        // the top-face carries of a column are split over its z-groups by field
        // (warp-uniform: the group index is the slowest thread coordinate)
        constexpr int NG = N / K;
        const bool carry_f = (MAIN && NG > 1) ? (more && (f % NG) == oz0 / K) : do_carry;
        if (carry_f) {
            double top = 0.0;
#pragma unroll
            for (int m = 0; m <= N; ++m) top = fma(sDx[N * (N + 1) + m], val[m], top);
            carw[f * (T::CYW * T::CXW)] = top;
        }
    };
    double R0[K], R1[K], R2[K], R3[K], R4[K], dwz[K], dPLz[K];
    {
        double gxv[K], gyv[K], gzv[K], divu[K];
        if (NEED_R) {
            grad(0, true, gxv, gyv, gzv);
#pragma unroll
            for (int k = 0; k < K; ++k) R0[k] = (u[k] * gxv[k] + v[k] * gyv[k]) + w[k] * gzv[k];
            grad(1, true, gxv, gyv, gzv);
#pragma unroll
            for (int k = 0; k < K; ++k) {
                R1[k] = (u[k] * gxv[k] + v[k] * gyv[k]) + w[k] * gzv[k];
                divu[k] = gxv[k];
            }
            grad(2, true, gxv, gyv, gzv);
#pragma unroll
            for (int k = 0; k < K; ++k) {
                R2[k] = (u[k] * gxv[k] + v[k] * gyv[k]) + w[k] * gzv[k];
                divu[k] += gyv[k];
            }
        }
        grad(3, NEED_R, gxv, gyv, gzv);
#pragma unroll
        for (int k = 0; k < K; ++k) dwz[k] = gzv[k];
        if (NEED_R) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                R3[k] = (u[k] * gxv[k] + v[k] * gyv[k]) + w[k] * gzv[k];
                divu[k] += gzv[k];
            }
            grad(4, true, gxv, gyv, gzv);
#pragma unroll
            for (int k = 0; k < K; ++k) R4[k] = (u[k] * gxv[k] + v[k] * gyv[k]) + w[k] * gzv[k];
            grad(5, true, gxv, gyv, gzv);   // grad P'
#pragma unroll
            for (int k = 0; k < K; ++k) {
                R1[k] += gxv[k] * rinv[k];
                R2[k] += gyv[k] * rinv[k];
                R3[k] += gzv[k] * rinv[k];
                R0[k] += rho[k] * divu[k];
            }
        }
        if (NEED_L) {
            grad(6, false, gxv, gyv, gzv);   // d/dz of the linearised pressure
#pragma unroll
            for (int k = 0; k < K; ++k) dPLz[k] = gzv[k];
        }
    }
    const double gr = a.ph.g;
    if (af_smem) {
        mbar_wait(mbaf, ez & 1);
#pragma unroll
        for (int k = 0; k < K; ++k)
#pragma unroll
            for (int f = 0; f < 5; ++f) {
                const int i = ((f * N + oz0 + k) * T::OYM + oy) * T::OX + ox;
                if (MODE == M_S2) Ain[k][f] = sAF[i];
                Fin[k][f] = sAF[T::AFB + i];
            }
    }
    const bool bx = (gx == 0) || (gx == g.X - 1);
    const bool by = g.slab || (gy == 0) || (gy == g.Y - 1);
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int gz = gzk[k];
        const double drho0 = LT[(gz) * T::NTAB + T_DRHO0];
        const double dth0 = LT[(gz) * T::NTAB + T_DTH0];
        const bool bz = (gz == 0) || (gz == g.Z - 1);
        double Rv[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        if (NEED_R) {
            const double theta = LT[(gz) * T::NTAB + T_TH0] + th[k];
            if (!(isfinite(r[k]) && isfinite(u[k]) && isfinite(v[k]) && isfinite(w[k]) &&
                  isfinite(th[k])))
                atomicOr(a.flags, HEVI_F_NONFINITE_IN(a.stage));
            if (!(rho[k] > 0.0) || !(theta > 0.0)) atomicOr(a.flags, HEVI_F_EOS(a.stage));
            // euler.nonlinear_rhs set2nc (euler.py:458-473), DSS folded into the derivatives;
            // euler.zero_normal_velocity after the DSS (euler.py:494-496)
            Rv[0] = -(R0[k] + w[k] * drho0);
            Rv[1] = bx ? 0.0 : -R1[k];
            Rv[2] = by ? 0.0 : -R2[k];
            Rv[3] = bz ? 0.0 : -(R3[k] + (r[k] * rinv[k]) * gr);
            Rv[4] = -(R4[k] + w[k] * dth0);
        }
        double Lv[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        if (NEED_L) {
            // euler.linear_operator(vertical_only=True), set2nc (euler.py:333-361)
            const double irho0 = LT[(gz) * T::NTAB + T_IRHO0];
            Lv[0] = -(w[k] * drho0 + LT[(gz) * T::NTAB + T_RHO0] * dwz[k]);
            Lv[3] = bz ? 0.0 : -(dPLz[k] * irho0 + (r[k] * irho0) * gr);
            Lv[4] = -(w[k] * dth0);
        }
        const long long oo = o[k];
        if (MODE == M_R) {
#pragma unroll
            for (int f = 0; f < 5; ++f) a.out[oo + f * fs] = Rv[f];
        } else if (MODE == M_L) {
#pragma unroll
            for (int f = 0; f < 5; ++f) a.out[oo + f * fs] = Lv[f];
        } else if (MODE == M_S1) {
            // imexcore.ark_imex_step (imexcore.py:398-403, 409-411)
            const double dt = a.dt;
            const double qv[5] = {r[k], u[k], v[k], w[k], th[k]};
            double pr[5];
#pragma unroll
            for (int f = 0; f < 5; ++f) {
                pr[f] = qv[f] + dt * (a.a_p * (Rv[f] - Lv[f]) + a.at_p * Lv[f]);
                a.A[oo + f * fs] = qv[f] + dt * (a.a_a * (Rv[f] - Lv[f]) + a.at_a * Lv[f]);
                a.F[oo + f * fs] = qv[f] + a.cb * Rv[f];
            }
            a.P[oo] = pr[0];
            a.P[oo + 3 * fs] = pr[3];
            a.P[oo + 4 * fs] = pr[4];
            a.Quv[oo + fs] = bx ? 0.0 : pr[1];
            a.Quv[oo + 2 * fs] = by ? 0.0 : pr[2];
        } else if (MODE == M_S2) {
            const double dt = a.dt;
            double pr[5];
#pragma unroll
            for (int f = 0; f < 5; ++f) {
                pr[f] = Ain[k][f] + dt * (a.a_p * (Rv[f] - Lv[f]) + a.at_p * Lv[f]);
                a.F[oo + f * fs] = Fin[k][f] + a.cb * Rv[f];
            }
            a.P[oo] = pr[0];
            a.P[oo + 3 * fs] = pr[3];
            a.P[oo + 4 * fs] = pr[4];
            a.Quv[oo + fs] = bx ? 0.0 : pr[1];
            a.Quv[oo + 2 * fs] = by ? 0.0 : pr[2];
        } else if (MODE == M_RK) {
            // SSP RK(5,3) Shu-Osher stage (imexcore.py:111-126)
            const double qv[5] = {r[k], u[k], v[k], w[k], th[k]};
            bool fin = true;
#pragma unroll
            for (int f = 0; f < 5; ++f) {
                double val = a.A ? a.a_p * Ain[k][f] : 0.0;
                val = val + a.at_p * qv[f];
                val = val + a.cb * Rv[f];
                fin = fin && isfinite(val);
                a.out[oo + f * fs] = val;
            }
            if (a.rk_final && !fin) atomicOr(a.flags, HEVI_F_NONFINITE_OUT);
        } else {
            bool fin = true;
#pragma unroll
            for (int f = 0; f < 5; ++f) {
                const double val = Fin[k][f] + a.cb * Rv[f];
                fin = fin && isfinite(val);
                a.out[oo + f * fs] = val;
            }
            if (!fin) atomicOr(a.flags, HEVI_F_NONFINITE_OUT);
        }
    }
}

// fallback staging without TMA: level z0 of the tile (+halo) into a ring
// slot, same placement (x shifted by xsh) and zero fill as the TMA
template <int N, int NY, int TX, int TY>
__device__ __forceinline__ void stage_level_manual(double* slot, const EArgs& a, int tx0, int ty0, int z0) {
    using T = E2<N, NY, TX, TY>;
    const Geo& g = a.g;
    constexpr int TOT = 5 * T::PL;
    for (int i = threadIdx.x; i < TOT; i += T::BLK) {
        const int x = i % T::LXT;
        const int t = i / T::LXT;
        const int y = t % T::LY;
        const int f = t / T::LY;
        const int ix = tx0 + x, iy = ty0 + y;
        double v = 0.0;
        if (ix >= 0 && ix < g.lX && iy >= 0 && iy < g.lY && z0 < g.Z)
            v = a.q[f * g.fs + ((long long)z0 * g.lY + iy) * g.px + ix];
        slot[i] = v;
    }
}

template <int N, int NY, int TX, int TY, int MODE, int MINB>
__global__ void __launch_bounds__(E2<N, NY, TX, TY>::BLK, MINB)
    k_explicit2(const EArgs a, const __grid_constant__ CUtensorMap tmap,
                const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmF,
                const __grid_constant__ CUtensorMap tmP) {
    using T = E2<N, NY, TX, TY>;
    constexpr int PL = T::PL, LXT = T::LXT, RING = T::RING, SS = T::SS, BLK = T::BLK;
    constexpr bool NEED_R = (MODE != M_L);
    extern __shared__ __align__(128) unsigned char smraw[];
    // TMA destinations must be 128-byte aligned: align the carve-up explicitly
    double* smd = reinterpret_cast<double*>(
        smraw + ((128u - ((unsigned)__cvta_generic_to_shared(smraw) & 127u)) & 127u));
    double* Sa = smd;                 // ring, 128-byte aligned slots (TMA destinations)
    double* sAF = Sa + T::S_N;        // [A | F] layer boxes (128-byte aligned)
    double* CAR = sAF + T::af_of(MODE);
    double* XF = CAR + T::CAR_N;
    double* sDx = XF + T::XF_N;
    double* sDy = sDx + T::DN;
    double* LT = sDy + T::DNY;
    uint64_t* mbar = reinterpret_cast<uint64_t*>(LT + T::NTAB * a.g.Z);   // [2] per layer parity, [2] A/F
    const Geo& g = a.g;
    const int Z = g.Z;
    const int tid = threadIdx.x;
    const int ex0 = g.ex_b + blockIdx.x * TX;
    const int ey0 = g.ey_b + blockIdx.y * TY;
    const int nxe = min(TX, g.ex_e - ex0);
    const int nye = min(TY, g.ey_e - ey0);
    const int oxn = nxe * N + ((ex0 + nxe == g.nex) ? 1 : 0);
    const int oyn = nye * NY + ((ey0 + nye == g.ney) ? 1 : 0);
    const int oxm = nxe * N;                                  // main x extent
    const int oym = nye * NY + (NY == 1 ? 1 : 0);             // main y extent
    const int gxlo = (ex0 - 1) * N, gylo = (ey0 - 1) * NY;

    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        mbar_init(&mbar[2], 1);
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
    }
    for (int i = tid; i < T::DN; i += BLK) sDx[i] = a.Dx[i];
    for (int i = tid; i < T::DNY; i += BLK) sDy[i] = a.Dy[i];
    for (int k = tid; k < Z; k += BLK) {
        LT[(k) * T::NTAB + T_RHO0] = a.lv.rho0[k];
        LT[(k) * T::NTAB + T_TH0] = a.lv.theta0[k];
        LT[(k) * T::NTAB + T_E0] = a.lv.E0[k];
        LT[(k) * T::NTAB + T_C0] = a.lv.c0[k];
        LT[(k) * T::NTAB + T_IRT0] = a.lv.irt0[k];
        LT[(k) * T::NTAB + T_G0] = a.lv.G0[k];
        LT[(k) * T::NTAB + T_H0] = a.lv.H0[k];
        LT[(k) * T::NTAB + T_DRHO0] = a.lv.drho0[k];
        LT[(k) * T::NTAB + T_DTH0] = a.lv.dth0[k];
        LT[(k) * T::NTAB + T_CZ] = a.cz[k];
        LT[(k) * T::NTAB + T_P0F] = a.lv.P0f[k];
        LT[(k) * T::NTAB + T_IRHO0] = 1.0 / a.lv.rho0[k];
    }
    __syncthreads();
    // window-local TMA coordinates of the tile origin
    const int txr = gxlo - g.x0, ty0 = gylo - g.y0;
    const int xsh = txr & 1;          // staged column of lx is lx + xsh
    const int tx0 = txr - xsh;
    double* S = Sa + xsh;             // compute view: column lx at S[... + lx]
    const bool use_tma = a.use_tma != 0;
    // P' of the stage input (stage 0: hevi_stage's k_pp_plane; stages 1, 2:
    // the column solve) arrives with each level (its own 1-field TMA) instead
    // of being formed here for every staged point
    const bool pp_tma = use_tma && a.pp_in != nullptr && (MODE == M_S1 || MODE == M_S2 || MODE == M_S3);
    const uint32_t lvl_bytes = T::LVL_BYTES + (pp_tma ? T::PP_BYTES : 0u);
    auto load_level = [&](int L, uint64_t* bar) {
        double* slot = Sa + (L % RING) * SS;
        tma_load_4d(slot, &tmap, bar, tx0, ty0, L, 0);
        if (pp_tma) tma_load_4d(slot + T::PPO, &tmP, bar, tx0, ty0, L, 0);
    };
    // layers 0 and 1 in flight before the sweep starts (levels 0..2N, slots 0..2N)
    if (use_tma && tid == 0) {
        mbar_expect_tx(&mbar[0], (N + 1) * lvl_bytes);
        for (int l = 0; l <= N; ++l) load_level(l, &mbar[0]);
        if (g.nez > 1) {
            mbar_expect_tx(&mbar[1], N * lvl_bytes);
            for (int l = N + 1; l <= 2 * N; ++l) load_level(l, &mbar[1]);
        }
    }

    // ---- the thread's main points (fixed for the whole sweep) -------------
    constexpr int K = T::K;
    const bool has_main = tid < T::NT;
    const int mox = tid % T::OX;
    const int moy = (tid / T::OX) % T::OYM;
    const int mop = tid / (T::OX * T::OYM);      // z-group: warp-uniform
    const int moz = mop * K;
    const bool main_ok = has_main && mox < oxm && moy < oym;
    const int mgx = ex0 * N + mox, mgy = ey0 * NY + moy;
    const PAx max_ = pax(mgx, mox + N, N, g.nex);
    const PAx may_ = pax(mgy, moy + NY, NY, g.ney);
    DRows<N, NY, K> Dm;
    double mcx = 0.0, mcy = 0.0;
    if (main_ok) {
#pragma unroll
        for (int m = 0; m <= N; ++m) {
            Dm.x[m] = sDx[max_.row * (N + 1) + m];
#pragma unroll
            for (int k = 0; k < K; ++k) Dm.z[k][m] = sDx[(moz + k) * (N + 1) + m];
        }
#pragma unroll
        for (int m = 0; m <= NY; ++m) Dm.y[m] = sDy[may_.row * (NY + 1) + m];
        mcx = __ldg(a.cx + mgx);
        mcy = __ldg(a.cy + mgy);
    }
    const double* bc = a.bc;

    // HEVI_PHASE_TIMING debug builds: per-phase clock64 sums (tools/phase_timing.py)
#ifdef HEVI_PHASE_TIMING
    unsigned long long tph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    unsigned long long t0 = clock64(), t1;
#define PH(i) do { t1 = clock64(); tph[i] += t1 - t0; t0 = t1; } while (0)
#else
#define PH(i) do { } while (0)
#endif
    const bool af_tma = T::AF_N > 0 && a.af_tma && ((HEVI_X_AFTMA_MASK >> MODE) & 1);
    for (int ez = 0; ez < g.nez; ++ez) {
        const int base = ez * N;
        if (af_tma && tid == 0) {
            // the previous layer's epilogue reads are ordered by its final barrier
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            const int ax0 = ex0 * N - g.x0, ay0 = ey0 * NY - g.y0;
            if (MODE == M_S2) {
                mbar_expect_tx(&mbar[2], 2 * T::AF_BYTES);
                tma_load_4d(sAF, &tmA, &mbar[2], ax0, ay0, base, 0);
            } else {
                mbar_expect_tx(&mbar[2], T::AF_BYTES);
            }
            tma_load_4d(sAF + T::AFB, &tmF, &mbar[2], ax0, ay0, base, 0);
        }
        // ---------------- 1. this layer's new levels, P' in place -----------
        const int lz0 = (ez == 0) ? 0 : 1;
        if (use_tma) {
            mbar_wait(&mbar[ez & 1], (ez >> 1) & 1);
        } else {
            for (int lz = lz0; lz <= N; ++lz)
                stage_level_manual<N, NY, TX, TY>(Sa + ((base + lz) % RING) * SS, a, tx0, ty0, base + lz);
            __syncthreads();
        }
        PH(0);
        if (NEED_R && !pp_tma) {
            const int nconv = (N + 1 - lz0) * T::LY * T::LX;
            for (int idx = tid; idx < nconv; idx += BLK) {
                const int lx = idx % T::LX;
                const int t = idx / T::LX;
                const int ly = t % T::LY;
                const int gz = base + lz0 + t / T::LY;
                double* sp = S + (gz % RING) * SS + ly * LXT + lx;
                const double* lt = LT + gz * T::NTAB;
                sp[T::PPO] = pprime(sp[0], sp[4 * PL], lt[T_RHO0], lt[T_TH0], lt[T_E0], lt[T_C0],
                                    lt[T_IRT0], lt[T_P0F], bc, a.ph);
            }
        }
        if ((HEVI_X_MERGE_MASK >> MODE) & 1) {
            // face partials of the 5 state fields need only the TMA data
            // (with the P' plane staged by TMA its face partials are formed here too)
            const int NXF5 = ((HEVI_X_XF6 && pp_tma) ? 6 : 5) * TX * T::OYM * N;
            for (int it = tid; it < NXF5; it += BLK) {
                const int oz = it % N;
                int t = it / N;
                const int oy = t % T::OYM;
                t /= T::OYM;
                const int ae = t % TX;
                const int f = t / TX;
                const double* sx = S + T::foff(f) + ((base + oz) % RING) * SS + (oy + NY) * LXT + ae * N;
                double s = 0.0;
#pragma unroll
                for (int m = 0; m <= N; ++m) s = fma(sDx[N * (N + 1) + m], sx[m], s);
                XF[it] = s;
            }
        }
        PH(1);
        __syncthreads();
        PH(2);
        // ---------------- 2. shared partial sums ----------------------------
        double* CARw = CAR + (ez & 1) * (7 * T::CYW * T::CXW);
        const double* CARr = CAR + ((ez + 1) & 1) * (7 * T::CYW * T::CXW);
        if (!((HEVI_X_MERGE_MASK >> MODE) & 1)) {
            // row N of the left element at the tile's element x-faces
            constexpr int NXF = T::XF_N;
            for (int it = tid; it < NXF; it += BLK) {
                const int oz = it % N;
                int t = it / N;
                const int oy = t % T::OYM;
                t /= T::OYM;
                const int ae = t % TX;
                const int f = t / TX;
                const double* sx = S + T::foff(f) + ((base + oz) % RING) * SS + (oy + NY) * LXT + ae * N;
                double s = 0.0;
#pragma unroll
                for (int m = 0; m <= N; ++m) s = fma(sDx[N * (N + 1) + m], sx[m], s);
                XF[it] = s;
            }
        }
        PH(3);
        if (!((HEVI_X_MERGE_MASK >> MODE) & 1)) __syncthreads();
        PH(4);
        // ---------------- 3. points ------------------------------------------
        if (main_ok) {
            e2_pts<N, NY, TX, TY, MODE, true, K>(a, S, CARr, CARw, XF, LT, Dm, sDx, sDy, max_, may_,
                                                 moz, mox, moy, mgx, mgy, ez, mcx, mcy, Z,
                                                 af_tma ? sAF : nullptr, &mbar[2], HEVI_X_XF6 && pp_tma);
        }
        // points outside the main box: domain-end x column / y row, top level
        const int ozn = N + ((ez == g.nez - 1) ? 1 : 0);
        const int nfull = oxn * oyn * ozn;
        if (nfull > oxm * oym * N) {
            for (int p = tid; p < nfull; p += BLK) {
                const int ox = p % oxn;
                const int t = p / oxn;
                const int oy = t % oyn;
                const int oz = t / oyn;
                if (ox < oxm && oy < oym && oz < N) continue;
                const int gx = ex0 * N + ox, gy = ey0 * NY + oy, gz = base + oz;
                const PAx ax = pax(gx, ox + N, N, g.nex);
                const PAx ay = pax(gy, oy + NY, NY, g.ney);
                const PAx az = pax(gz, oz, N, g.nez);
                DRows<N, NY, 1> De;
#pragma unroll
                for (int m = 0; m <= N; ++m) {
                    De.x[m] = sDx[ax.row * (N + 1) + m];
                    De.z[0][m] = sDx[az.row * (N + 1) + m];
                }
#pragma unroll
                for (int m = 0; m <= NY; ++m) De.y[m] = sDy[ay.row * (NY + 1) + m];
                e2_pts<N, NY, TX, TY, MODE, false, 1>(a, S, CARr, CARw, XF, LT, De, sDx, sDy, ax, ay,
                                                      oz, ox, oy, gx, gy, ez, __ldg(a.cx + gx),
                                                      __ldg(a.cy + gy), Z);
            }
        }
        PH(5);
        __syncthreads();
        PH(6);
        // levels base .. base+N-1 are dead: refill their slots with layer ez+2
        if (use_tma && tid == 0 && ez + 2 < g.nez) {
            // generic-proxy accesses of the slots are ordered before the async-proxy refill
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&mbar[ez & 1], N * lvl_bytes);
            for (int l = 1; l <= N; ++l) load_level(base + 2 * N + l, &mbar[ez & 1]);
        }
    }
#ifdef HEVI_PHASE_TIMING
    if (a.dbg) {
        for (int i = 0; i < 7; ++i) atomicAdd(a.dbg + i, tph[i]);
        atomicAdd(a.dbg + 7, 1ull);
    }
#endif
#undef PH
}
