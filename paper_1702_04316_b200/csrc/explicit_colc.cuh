// explicit_colc.cuh -- column-sweep explicit kernel for the conservative set
// set2c on 3D boxes, N = 4 (included by hevi.cu after explicit_col.cuh).
//
// euler.nonlinear_rhs set2c (euler.py:474-487) is a flux form,
//   R = -( div U,  div(U_m U / rho + P' e_m) + rho' g e_z,  div(theta U) ),
// with theta = Theta / rho and P' = EOS(rho, theta) - P0f; L_V set2c
// (euler.py:350-361).  With the DSS folded into the derivatives (hevi.cu)
// each point needs
//   d/dx of  U, UU/rho+P', UV/rho, UW/rho, theta U        (5 x-quantities)
//   d/dy of  V, UV/rho, VV/rho+P', VW/rho, theta V        (5 y-quantities)
//   d/dz of  W, UW/rho, VW/rho, WW/rho+P', theta W, F0 Theta'   (6 z-quantities)
// The structure is k_ecol's (tile 4x4 elements, one thread per column, TMA
// level ring, register z-window, face partials, A/F ring, fused epilogues);
// what set2c adds is a convert phase: for the next level every staged point
// forms 1/rho, theta, P' (binomial series in Theta'/Theta0: rho theta =
// Theta) and the 7 flux-product planes the x/y lines read, into a double
// buffer.  The z-window holds the 6 z-quantities of the column's element
// layer, formed from the raw fields at the layer start.  Two barriers per
// level (convert -> faces -> next level).
#pragma once

template <int N, int MODE>
struct ECC {
    static constexpr int TX = 4, TY = 4;
    static constexpr int OX = TX * N, OY = TY * N, BLK = OX * OY;
    static constexpr int LX = OX + N + 1, LY = OY + N + 1;
    static constexpr int LXT = (LX + 1) / 2 * 2, PL = LXT * LY;
    static constexpr int SS = (5 * PL + 15) / 16 * 16;        // raw rho', U, V, W, Theta'
    static constexpr int NPB = 7;                              // flux-product planes
    static constexpr int PBS = (NPB * PL + 15) / 16 * 16;      // one level's products (128-byte aligned)
    static constexpr int NAF = (MODE == M_S2) ? 2 : (MODE == M_S3) ? 1 : 0;
    static constexpr int SAF = NAF ? 2 : 0;
    static constexpr int SAFM = NAF ? SAF : 1;
    static constexpr int AFB = 5 * OX * OY;
    static constexpr int S = 6;
    static constexpr int NXF = 5 * OY * TX, NYF = 5 * TY * OX;
    static constexpr int DN = (N + 1) * (N + 1);
    static constexpr size_t SMEM =
        sizeof(double) * ((size_t)S * SS + 2 * PBS + (size_t)SAF * NAF * AFB + 2 * (NXF + NYF) + 2 * DN +
                          OX + OY) +
        sizeof(uint64_t) * (S + SAF) + 128;
    static constexpr uint32_t LVL_BYTES = (uint32_t)(sizeof(double) * 5 * PL);
    static constexpr uint32_t AF_BYTES = (uint32_t)(sizeof(double) * AFB);
};

// P' of set2c about the background: P = P0 (R Theta / P0)^gamma, delta =
// Theta'/Theta0; the level's constants and the short series' coefficients
// are hoisted (PPc), the rare wide branch is out of line with scalar args
struct PPc {
    double ith0, pb, c0;
    double b[6];
};

__device__ __forceinline__ PPc ecc_ppc(const EArgs& a, const LvlTab& lt, int gz) {
    PPc c;
    c.ith0 = lt.v[C_ITH0][gz];
    c.pb = lt.v[C_PB][gz];
    c.c0 = lt.v[C_C0][gz];
#pragma unroll
    for (int k = 0; k < 6; ++k) c.b[k] = a.bc[k];
    return c;
}

__device__ __noinline__ double ecc_pprime_wide(const EArgs& a, const LvlTab& lt, int gz, double delta,
                                               double rho, double Th) {
    if (fabs(delta) <= 0.125) {
        double s = a.bc[14];
#pragma unroll
        for (int k = 13; k >= 0; --k) s = fma(s, delta, a.bc[k]);
        return fma(lt.v[C_PB][gz], s * delta, lt.v[C_C0][gz]);
    }
    const double theta = (lt.v[C_TH0C][gz] + Th) / rho;
    return a.ph.P0 * pow(rho * a.ph.R * theta / a.ph.P0, a.ph.gamma) - lt.v[C_P0F][gz];
}

__device__ __forceinline__ double ecc_pprime(const EArgs& a, const LvlTab& lt, int gz, const PPc& c, double rho,
                                             double Th) {
    const double delta = Th * c.ith0;
    if (HEVI_PP_SHORT && fabs(delta) <= 0x1p-10) {
        double s = c.b[5];
#pragma unroll
        for (int k = 4; k >= 0; --k) s = fma(s, delta, c.b[k]);
        return fma(c.pb, s * delta, c.c0);
    }
    return ecc_pprime_wide(a, lt, gz, delta, rho, Th);
}

__device__ __forceinline__ double ecc_pprime(const EArgs& a, const LvlTab& lt, int gz, double rho, double Th) {
    return ecc_pprime(a, lt, gz, ecc_ppc(a, lt, gz), rho, Th);
}

// R, L_V of set2c at a point from its 16 derivative values (euler.py:481-487, 350-361)
template <int MODE>
__device__ __forceinline__ void ecc_finish(const double (&gx)[5], const double (&gy)[5], const double (&gz)[6],
                                           double r, double W, double th0, double dth0, double gr, bool bx, bool by,
                                           bool bz, double (&Rv)[5], double (&Lv)[5]) {
    constexpr bool NEED_L = (MODE == M_S1 || MODE == M_S2);
#pragma unroll
    for (int f = 0; f < 5; ++f) Rv[f] = Lv[f] = 0.0;
    Rv[0] = -((gx[0] + gy[0]) + gz[0]);
    Rv[1] = bx ? 0.0 : -((gx[1] + gy[1]) + gz[1]);
    Rv[2] = by ? 0.0 : -((gx[2] + gy[2]) + gz[2]);
    Rv[3] = bz ? 0.0 : -((gx[3] + gy[3]) + gz[3]) - r * gr;
    Rv[4] = -((gx[4] + gy[4]) + gz[4]);
    if (NEED_L) {
        Lv[0] = -gz[0];
        Lv[3] = bz ? 0.0 : -(gz[5] + r * gr);
        Lv[4] = -(th0 * gz[0] + W * dth0);
    }
}

template <int N, int MODE>
__global__ void __launch_bounds__(ECC<N, MODE>::BLK, 1)
    k_ecolc(const EArgs a, const __grid_constant__ LvlTab lt, const __grid_constant__ CUtensorMap tmq,
            const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmF) {
    using T = ECC<N, MODE>;
    constexpr int PL = T::PL, LXT = T::LXT, SS = T::SS, S = T::S, BLK = T::BLK;
    constexpr int OX = T::OX, OY = T::OY, TX = T::TX, TY = T::TY, LY = T::LY;
    constexpr bool NEED_L = (MODE == M_S1 || MODE == M_S2);
    static_assert(N == 4, "x-line vector loads assume N = 4");
    static_assert(MODE == M_R || MODE == M_S1 || MODE == M_S2 || MODE == M_S3, "stage kernels and R");
    extern __shared__ __align__(128) unsigned char smraw[];
    double* ring = reinterpret_cast<double*>(
        smraw + ((128u - ((unsigned)__cvta_generic_to_shared(smraw) & 127u)) & 127u));
    double* PB = ring + S * SS;                        // [2][PBS]: the 7 flux-product planes of a level
    double* sAF = PB + 2 * T::PBS;                     // [SAF][NAF][5][OY][OX] (TMA destinations)
    double* XFb = sAF + T::SAF * T::NAF * T::AFB;      // [2][NXF]
    double* YFb = XFb + 2 * T::NXF;                    // [2][NYF]
    double* sD = YFb + 2 * T::NYF;
    double* sC = sD + 2 * T::DN;
    uint64_t* mbar = reinterpret_cast<uint64_t*>(sC + OX + OY);

    const Geo& g = a.g;
    const int Z = g.Z;
    const int tid = threadIdx.x;
    const int ox = tid % OX, oy = tid / OX;
    int bxt, byt;
    ec_tile(a, bxt, byt);
    const int ex0 = g.ex_b + bxt * TX, ey0 = g.ey_b + byt * TY;
    const int gx = ex0 * N + ox, gy = ey0 * N + oy;
    const bool own = gx < g.ex_e * N && gy < g.ey_e * N;
    const int tx0 = (ex0 - 1) * N - g.x0, ty0 = (ey0 - 1) * N - g.y0;

    if (HEVI_EDGE_PDL_C) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // see k_ecol
    if (tid == 0) {
        for (int s = 0; s < S + T::SAF; ++s) mbar_init(&mbar[s], 1);
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmq) : "memory");
    }
    for (int i = tid; i < T::DN; i += BLK) {
        sD[i] = a.Dx[i];
        sD[T::DN + i] = a.Dy[i];
    }
    if (tid < OX) sC[tid] = (ex0 * N + tid < g.X) ? a.cx[ex0 * N + tid] : 0.0;
    else if (tid < OX + OY) sC[tid] = (ey0 * N + tid - OX < g.Y) ? a.cy[ey0 * N + tid - OX] : 0.0;
    __syncthreads();
    auto issue = [&](int l) {
        double* slot = ring + (l % S) * SS;
        uint64_t* bar = &mbar[l % S];
        mbar_expect_tx(bar, T::LVL_BYTES);
        tma_load_4d(slot, &tmq, bar, tx0, ty0, l, 0);
    };
    const int ax0 = ex0 * N - g.x0, ay0 = ey0 * N - g.y0;
    auto issue_af = [&](int l) {
        if (T::NAF == 0) return;
        double* dst = sAF + (l % T::SAFM) * (T::NAF * T::AFB);
        uint64_t* bar = &mbar[S + l % T::SAFM];
        mbar_expect_tx(bar, T::NAF * T::AF_BYTES);
        if (MODE == M_S2) {
            tma_load_4d(dst, &tmA, bar, ax0, ay0, l, 0);
            tma_load_4d(dst + T::AFB, &tmF, bar, ax0, ay0, l, 0);
        } else {
            tma_load_4d(dst, &tmF, bar, ax0, ay0, l, 0);
        }
    };
    if (tid == 0) {
        for (int l = 0; l < S && l < Z; ++l) issue(l);
        for (int l = 0; l < T::SAF && l < Z; ++l) issue_af(l);
    }

    const int rx = ox % N, ry = oy % N;
    const double cxv = own ? sC[ox] : 0.0, cyv = own ? sC[OX + oy] : 0.0;
    double Dxr[N + 1], Dyr[N + 1];
#pragma unroll
    for (int m = 0; m <= N; ++m) {
        Dxr[m] = cxv * sD[rx * (N + 1) + m];
        Dyr[m] = cyv * sD[T::DN + ry * (N + 1) + m];
    }
    // element-face weights; the domain's low walls (gx = 0, gy = 0) have no lower element
    const double fxs = (rx == 0 && gx > 0) ? cxv : 0.0, fys = (ry == 0 && gy > 0) ? cyv : 0.0;
    const bool bx = (gx == 0), by = (gy == 0);
    const int lx = ox + N, ly = oy + N;
    const int xo = ly * LXT + (lx - rx);
    const int yo = (ly - ry) * LXT + lx;
    const int po = ly * LXT + lx;
    const int xfo = oy * TX + ox / N;
    const int yfo = (oy / N) * OX + ox;
    const long long colo = (long long)(gy - g.y0) * g.px + (gx - g.x0);
    const long long zs = (long long)g.lY * g.px;
    const double gr = a.ph.g;

    // x-quantity q: U (raw) or products 0 UU/rho+P', 1 UV/rho, 2 UW/rho, 3 theta U;
    // y-quantity q: V (raw) or products 1 UV/rho, 4 VV/rho+P', 5 VW/rho, 6 theta V
    auto xplane = [&](int q, const double* slot, const double* pb) -> const double* {
        return q == 0 ? slot + PL : pb + (q - 1) * PL;
    };
    auto yplane = [&](int q, const double* slot, const double* pb) -> const double* {
        return q == 0 ? slot + 2 * PL : pb + (q == 1 ? 1 : q + 2) * PL;
    };

    // convert phase: flux products of level l at every staged point
    auto convert = [&](int l) {
        const double* slot = ring + (l % S) * SS;
        double* pb = PB + (l & 1) * T::PBS;
        const double rho0 = lt.v[C_RHO0][l], Th0 = lt.v[C_TH0C][l];
        const PPc ppc = ecc_ppc(a, lt, l);
        static_assert(LY * LXT <= 2 * BLK, "convert: two passes over the staged plane");
#pragma unroll
        for (int i = tid; i < LY * LXT; i += BLK) {
            const double r = slot[i], U = slot[PL + i], V = slot[2 * PL + i], W = slot[3 * PL + i],
                         Th = slot[4 * PL + i];
            const double rho = rho0 + r;
            const double irho = 1.0 / rho;
            const double theta = (Th0 + Th) * irho;
            const double pp = ecc_pprime(a, lt, l, ppc, rho, Th);
            pb[0 * PL + i] = (U * U) * irho + pp;
            pb[1 * PL + i] = (U * V) * irho;
            pb[2 * PL + i] = (U * W) * irho;
            pb[3 * PL + i] = theta * U;
            pb[4 * PL + i] = (V * V) * irho + pp;
            pb[5 * PL + i] = (V * W) * irho;
            pb[6 * PL + i] = theta * V;
        }
    };
    // element-face partials of the 5 x- and 5 y-quantities of level l
    auto faces = [&](int l, int buf) {
        const double* slot = ring + (l % S) * SS;
        const double* pb = PB + (l & 1) * T::PBS;
        double* xf = XFb + buf * T::NXF;
        double* yf = YFb + buf * T::NYF;
        static_assert(T::NXF + T::NYF <= 3 * BLK, "faces: three passes");
#pragma unroll
        for (int i = tid; i < T::NXF + T::NYF; i += BLK) {
            if (i < T::NXF) {
                const int q = i / (OY * TX), rem = i % (OY * TX);
                const int yy = rem / TX, j = rem % TX;
                const double* s = xplane(q, slot, pb) + (yy + N) * LXT + j * N;
                double d = lt.dx[N * (N + 1)] * s[0];
#pragma unroll
                for (int m = 1; m <= N; ++m) d = fma(lt.dx[N * (N + 1) + m], s[m], d);
                xf[i] = d;
            } else {
                const int ii = i - T::NXF;
                const int q = ii / (TY * OX), rem = ii % (TY * OX);
                const int j = rem / OX, xx = rem % OX;
                const double* s = yplane(q, slot, pb) + (j * N) * LXT + xx + N;
                double d = lt.dy[N * (N + 1)] * s[0];
#pragma unroll
                for (int m = 1; m <= N; ++m) d = fma(lt.dy[N * (N + 1) + m], s[m * LXT], d);
                yf[ii] = d;
            }
        }
    };

    // z-window: W, UW/rho, VW/rho, WW/rho + P', theta W, F0 Theta' on levels base .. base+N
    double Wz[6][N + 1];
    double car[6];
#pragma unroll
    for (int f = 0; f < 6; ++f) {
        car[f] = 0.0;
#pragma unroll
        for (int m = 0; m <= N; ++m) Wz[f][m] = 0.0;
    }

    mbar_wait(&mbar[0], 0);
    convert(0);
    __syncthreads();
    faces(0, 0);
    __syncthreads();

    unsigned fl = 0;
    // one level of the sweep (KK: the level's row in the z-window, N on the top level)
    auto level = [&](const int l, auto kc) {
        constexpr int KK = decltype(kc)::v;   // -1: a rolled loop (row from the slot)
        const bool top = (KK == N) || (KK < 0 && l == Z - 1);
        const double* slot = ring + (l % S) * SS;
        const double* pb = PB + (l & 1) * T::PBS;
        const double* xfb = XFb + (l & 1) * T::NXF;
        const double* yfb = YFb + (l & 1) * T::NYF;
        double dzr[N + 1];
#pragma unroll
        for (int m = 0; m <= N; ++m) dzr[m] = lt.dzs[l][m];
        const double czf = lt.czf[l];
        const double r = slot[po], U = slot[PL + po], V = slot[2 * PL + po], W = KK >= 0 ? Wz[0][KK < 0 ? 0 : KK] : slot[3 * PL + po],
                     Th = slot[4 * PL + po];
        double gxq[5], gyq[5], gzq[6];
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            const double* sx = xplane(q, slot, pb);
            const double2 v01 = *reinterpret_cast<const double2*>(sx + xo);
            const double2 v23 = *reinterpret_cast<const double2*>(sx + xo + 2);
            double dx = Dxr[0] * v01.x;
            dx = fma(Dxr[1], v01.y, dx);
            dx = fma(Dxr[2], v23.x, dx);
            dx = fma(Dxr[3], v23.y, dx);
            dx = fma(Dxr[4], sx[xo + 4], dx);
            gxq[q] = fma(fxs, xfb[q * (OY * TX) + xfo], dx);
            const double* sy = yplane(q, slot, pb);
            double dy = Dyr[0] * sy[yo];
#pragma unroll
            for (int m = 1; m <= N; ++m) dy = fma(Dyr[m], sy[yo + m * LXT], dy);
            gyq[q] = fma(fys, yfb[q * (TY * OX) + yfo], dy);
        }
#pragma unroll
        for (int f = 0; f < 6; ++f) {
            if (f == 5 && !NEED_L) {
                gzq[5] = 0.0;
                continue;
            }
            double dz = dzr[0] * Wz[f][0];
#pragma unroll
            for (int m = 1; m <= N; ++m) dz = fma(dzr[m], Wz[f][m], dz);
            gzq[f] = fma(czf, car[f], dz);
        }
        {
            // every thread computes; only owned points store or raise flags
            // (branch-free bits, one atomic per thread at the end)
            const double rho = lt.v[C_RHO0][l] + r;
            const double Theta = lt.v[C_TH0C][l] + Th;
            const double zc = fma(r, 0.0, fma(U, 0.0, fma(V, 0.0, fma(W, 0.0, Th * 0.0))));
            unsigned b = (zc == zc) ? 0u : HEVI_F_NONFINITE_IN(a.stage);
            b |= (rho > 0.0 && Theta / rho > 0.0) ? 0u : HEVI_F_EOS(a.stage);
            fl |= own ? b : 0u;
            double Ai[5] = {0, 0, 0, 0, 0}, Fi[5] = {0, 0, 0, 0, 0};
            if (T::NAF) {
                mbar_wait(&mbar[S + l % T::SAFM], (l / T::SAFM) & 1);
                const double* af = sAF + (l % T::SAFM) * (T::NAF * T::AFB) + tid;
#pragma unroll
                for (int f = 0; f < 5; ++f) {
                    if (MODE == M_S2) {
                        Ai[f] = af[f * OX * OY];
                        Fi[f] = af[T::AFB + f * OX * OY];
                    } else {
                        Fi[f] = af[f * OX * OY];
                    }
                }
            }
            double Rv[5], Lv[5];
            ecc_finish<MODE>(gxq, gyq, gzq, r, W, lt.v[C_TH0][l], lt.v[C_DTH0][l], gr, bx, by, (l == 0) || top,
                             Rv, Lv);
            PtSt p;
            p.r = r;
            p.u = U;
            p.v = V;
            p.w = W;
            p.th = Th;
            ec_epilogue<MODE>(a, lt, colo + (long long)l * zs, l, p, Rv, Lv, Ai, Fi, bx, by, own, &fl);
        }
        if (l + 1 < Z) convert(l + 1);
        __syncthreads();
        if (l + 1 < Z) faces(l + 1, (l + 1) & 1);
        __syncthreads();
        if (tid == 32 * (l % (BLK / 32))) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (l + S < Z) issue(l + S);
            if (T::NAF && l + T::SAF < Z) issue_af(l + T::SAF);
        }
    };
    // the z-window of the element layer starting at level l (levels l .. l+N)
    auto zwin = [&](const int l) {
        if (l > 0) {
#pragma unroll
            for (int f = 0; f < 6; ++f) {
                double c = lt.dz[N * (N + 1)] * Wz[f][0];
#pragma unroll
                for (int m = 1; m <= N; ++m) c = fma(lt.dz[N * (N + 1) + m], Wz[f][m], c);
                car[f] = c;
            }
        }
#pragma unroll
        for (int m = 1; m <= N; ++m) mbar_wait(&mbar[(l + m) % S], ((l + m) / S) & 1);
#pragma unroll
        for (int m = 0; m <= N; ++m) {
            const double* sp = ring + ((l + m) % S) * SS + po;
            const double r = sp[0], U = sp[PL], V = sp[2 * PL], W = sp[3 * PL], Th = sp[4 * PL];
            const double rho = lt.v[C_RHO0][l + m] + r;
            const double irho = 1.0 / rho;
            const double theta = (lt.v[C_TH0C][l + m] + Th) * irho;
            Wz[0][m] = W;
            Wz[1][m] = (U * W) * irho;
            Wz[2][m] = (V * W) * irho;
            Wz[3][m] = (W * W) * irho + ecc_pprime(a, lt, l + m, rho, Th);
            Wz[4][m] = theta * W;
            Wz[5][m] = lt.v[C_F0C][l + m] * Th;
        }
    };
    if (MODE == M_S1) {
        // rolled (unrolled, stage 0 rises from 228 to 240 registers and slows by 3 %)
        int k = 0;
        for (int l = 0; l < Z; ++l) {
            const bool last = (l == Z - 1);
            if (k == 0 && !last) zwin(l);
            level(l, KI<-1>{});
            if (!last) k = (k + 1 == N) ? 0 : k + 1;
        }
    } else {
        // element layers, unrolled: the own point's W is window row KK
        for (int l0 = 0; l0 + 1 < Z; l0 += N) {
            zwin(l0);
            level(l0, KI<0>{});
            level(l0 + 1, KI<1>{});
            level(l0 + 2, KI<2>{});
            level(l0 + 3, KI<3>{});
        }
        level(Z - 1, KI<N>{});
    }
    if (fl) atomicOr(a.flags, fl);
}

// set2c domain-end planes: one thread per point, the quantities formed per
// line node from global memory
template <int N, int MODE>
__global__ void __launch_bounds__(128) k_ecolc_edge(const EArgs a, const __grid_constant__ LvlTab lt, int nxc,
                                                    int nyr, int xlo, int ylo) {
    constexpr bool NEED_L = (MODE == M_S1 || MODE == M_S2);
    const Geo& G = a.g;
    const long long per = (long long)nxc + nyr;
    const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= per * G.Z) return;
    const int gz = (int)(id / per);
    const int cc = (int)(id % per);
    int gx, gy;
    if (cc < nxc) {
        gx = G.X - 1;
        gy = ylo + cc;
    } else {
        gx = xlo + (cc - nxc);
        gy = G.Y - 1;
    }
    const long long fs = G.fs, zs = (long long)G.lY * G.px;
    const int ix = gx - G.x0, iy = gy - G.y0;
    const long long o = (long long)gz * zs + (long long)iy * G.px + ix;
    const double* q = a.q;
    // quantity `k` (0..15: 5 x-, 5 y-, 6 z-quantities) at lattice offset off, level lz
    auto quant = [&](int kq, long long off, int lz) -> double {
        const double r = q[off], U = q[off + fs], V = q[off + 2 * fs], W = q[off + 3 * fs], Th = q[off + 4 * fs];
        const double rho = lt.v[C_RHO0][lz] + r;
        const double irho = 1.0 / rho;
        const double theta = (lt.v[C_TH0C][lz] + Th) * irho;
        switch (kq) {
            case 0: return U;
            case 1: return (U * U) * irho + ecc_pprime(a, lt, lz, rho, Th);
            case 2: return (U * V) * irho;
            case 3: return (U * W) * irho;
            case 4: return theta * U;
            case 5: return V;
            case 6: return (U * V) * irho;
            case 7: return (V * V) * irho + ecc_pprime(a, lt, lz, rho, Th);
            case 8: return (V * W) * irho;
            case 9: return theta * V;
            case 10: return W;
            case 11: return (U * W) * irho;
            case 12: return (V * W) * irho;
            case 13: return (W * W) * irho + ecc_pprime(a, lt, lz, rho, Th);
            case 14: return theta * W;
            default: return lt.v[C_F0C][lz] * Th;
        }
    };
    auto axis = [](int gi, int ne, int& row, int& s0, bool& face) {
        if (gi == ne * N) {
            row = N;
            s0 = gi - N;
            face = false;
        } else {
            row = gi % N;
            s0 = gi - row;
            face = (row == 0) && (gi > 0);
        }
    };
    int rxw, sx, ryw, sy, rzw, sz;
    bool fx, fy, fz;
    axis(gx, G.nex, rxw, sx, fx);
    axis(gy, G.ney, ryw, sy, fy);
    axis(gz, G.nez, rzw, sz, fz);
    const double cxv = __ldg(a.cx + gx), cyv = __ldg(a.cy + gy), czv = lt.v[C_CZ][gz];
    auto line = [&](int kq, int dir) -> double {
        double d = 0.0;
        if (dir == 0) {
            for (int m = 0; m <= N; ++m)
                d = fma(lt.dx[rxw * (N + 1) + m], quant(kq, o + (sx + m - gx), gz), d);
            if (fx) {
                double e = 0.0;
                for (int m = 0; m <= N; ++m) e = fma(lt.dx[N * (N + 1) + m], quant(kq, o + (gx - N + m - gx), gz), e);
                d += e;
            }
            return cxv * d;
        }
        if (dir == 1) {
            for (int m = 0; m <= N; ++m)
                d = fma(lt.dy[ryw * (N + 1) + m], quant(kq, o + (long long)(sy + m - gy) * G.px, gz), d);
            if (fy) {
                double e = 0.0;
                for (int m = 0; m <= N; ++m)
                    e = fma(lt.dy[N * (N + 1) + m], quant(kq, o + (long long)(m - N) * G.px, gz), e);
                d += e;
            }
            return cyv * d;
        }
        for (int m = 0; m <= N; ++m)
            d = fma(lt.dz[rzw * (N + 1) + m], quant(kq, o + (long long)(sz + m - gz) * zs, sz + m), d);
        if (fz) {
            double e = 0.0;
            for (int m = 0; m <= N; ++m)
                e = fma(lt.dz[N * (N + 1) + m], quant(kq, o + (long long)(m - N) * zs, gz - N + m), e);
            d += e;
        }
        return czv * d;
    };
    double gxq[5], gyq[5], gzq[6];
    for (int qq = 0; qq < 5; ++qq) {
        gxq[qq] = line(qq, 0);
        gyq[qq] = line(5 + qq, 1);
    }
    for (int qq = 0; qq < 6; ++qq) gzq[qq] = (qq == 5 && !NEED_L) ? 0.0 : line(10 + qq, 2);
    const double r = q[o], U = q[o + fs], V = q[o + 2 * fs], W = q[o + 3 * fs], Th = q[o + 4 * fs];
    const double rho = lt.v[C_RHO0][gz] + r, Theta = lt.v[C_TH0C][gz] + Th;
    if (!(isfinite(r) && isfinite(U) && isfinite(V) && isfinite(W) && isfinite(Th)))
        atomicOr(a.flags, HEVI_F_NONFINITE_IN(a.stage));
    if (!(rho > 0.0) || !(Theta / rho > 0.0)) atomicOr(a.flags, HEVI_F_EOS(a.stage));
    const bool bx = (gx == 0) || (gx == G.X - 1);
    const bool by = (gy == 0) || (gy == G.Y - 1);
    const bool bz = (gz == 0) || (gz == G.Z - 1);
    double Rv[5], Lv[5];
    ecc_finish<MODE>(gxq, gyq, gzq, r, W, lt.v[C_TH0][gz], lt.v[C_DTH0][gz], a.ph.g, bx, by, bz, Rv, Lv);
    double Ai[5] = {0, 0, 0, 0, 0}, Fi[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int f = 0; f < 5; ++f) {
        if (MODE == M_S2) Ai[f] = a.A[o + f * fs];
        if (MODE == M_S2 || MODE == M_S3) Fi[f] = a.F[o + f * fs];
    }
    PtSt p;
    p.r = r;
    p.u = U;
    p.v = V;
    p.w = W;
    p.th = Th;
    ec_epilogue<MODE>(a, lt, o, gz, p, Rv, Lv, Ai, Fi, bx, by);
    ec_edge_done();
}
