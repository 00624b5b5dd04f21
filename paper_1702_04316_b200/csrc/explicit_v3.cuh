// explicit_v3.cuh -- line-phase explicit-stage kernel (included by hevi.cu
// inside its anonymous namespace, after explicit_v2.cuh).
//
// Same sweep, TMA staging, level ring and P' series as v2, but the work of a
// layer is split into phases whose items register-block one element LINE:
//   X: item = (element x-line, row, level, field group): loads the line of
//      its fields once, forms the raw derivative sums at all N+1 line
//      positions ((N+1)^2 FMAs, N+1 loads per field) and turns them into
//      contributions to R (affine in the gradient, so contributions of the
//      two elements meeting at a face simply add): own points -> ACC,
//      the next element's face point -> FX;
//   Y: the same along y (ACC +=, FY);
//   Z: item = (column, field group) over the layer's z-line: own levels ->
//      ACC +=, row N -> the carry into the next layer's bottom face;
//   F: one thread per owned point: pointwise terms, no-flux projection,
//      flags, ARK2 stage epilogue (A/F prefetched one layer ahead).
// Every phase needs few registers, so the CTA runs 512 threads; each (point,
// component) accumulator has exactly one writer per phase (deterministic).
#pragma once

template <int N, int NY, int TX, int TY>
struct E3 {
    static constexpr int OX = TX * N, OY = TY * NY;
    static constexpr int EX = OX + 1, EY = OY + 1;            // extended owned box (domain ends)
    static constexpr int NZL = N + 1;                         // levels incl. the last layer's top
    static constexpr int LX = OX + N + 1, LXT = (LX + 2) / 2 * 2, LY = OY + NY + 1;
    static constexpr int NL = N + 1, PL = LY * LXT;
    static constexpr int BLK = 512;
    static constexpr int NPT = NZL * EY * EX;                 // extended points per layer
    static constexpr int NMAIN = OX * OY * N;                 // main points (one per thread)
    static constexpr int STG_N = 5 * NL * PL;
    static constexpr int S_N = 6 * NL * PL;                   // rho', u, v, w, theta', P'
    static constexpr int NACC = 7;                            // R0..R4, L0, L3 partials
    static constexpr int ACC_N = NACC * NPT;
    static constexpr int FX_N = 5 * NZL * EY * (TX + 1);
    static constexpr int FY_N = 5 * NZL * EX * (TY + 1);
    static constexpr int CAR_N = 2 * 7 * EY * EX;
    static constexpr int DN = (N + 1) * (N + 1), DNY = (NY + 1) * (NY + 1);
    static constexpr int NTAB = 12;
    static constexpr int CONV_N = N * LY * LX;
    static constexpr int CONV_IT = (CONV_N + BLK - 1) / BLK;
    static constexpr size_t fixed_bytes() {
        return sizeof(double) *
                   (size_t)(STG_N + S_N + ACC_N + FX_N + FY_N + CAR_N + DN + DNY + 1) + 128;
    }
    static constexpr uint32_t TMA_BYTES = (uint32_t)(sizeof(double) * STG_N);
    static_assert(NMAIN <= BLK, "one main point per thread");
};

template <int N, int NY, int TX, int TY>
__device__ __forceinline__ void stage_manual3(double* STG, const EArgs& a, int tx0, int ty0, int z0) {
    using T = E3<N, NY, TX, TY>;
    const Geo& g = a.g;
    constexpr int TOT = 5 * T::NL * T::LY * T::LXT;
    for (int i = threadIdx.x; i < TOT; i += T::BLK) {
        const int x = i % T::LXT;
        int t = i / T::LXT;
        const int y = t % T::LY;
        t /= T::LY;
        const int z = t % T::NL;
        const int f = t / T::NL;
        const int ix = tx0 + x, iy = ty0 + y, iz = z0 + z;
        double v = 0.0;
        if (ix >= 0 && ix < g.lX && iy >= 0 && iy < g.lY && iz < g.Z)
            v = a.q[f * g.fs + ((long long)iz * g.lY + iy) * g.px + ix];
        STG[i] = v;
    }
}

template <int N, int NY, int TX, int TY, int MODE>
__global__ void __launch_bounds__(512, 1)
    k_explicit3(const EArgs a, const __grid_constant__ CUtensorMap tmap) {
    using T = E3<N, NY, TX, TY>;
    constexpr int PL = T::PL, LXT = T::LXT, NL = T::NL, BLK = T::BLK;
    constexpr int EX = T::EX, EY = T::EY, NZL = T::NZL, NPT = T::NPT;
    constexpr int SF = NL * PL;                                // field stride in S / STG
    constexpr bool NEED_L = (MODE == M_L || MODE == M_S1 || MODE == M_S2);
    constexpr bool NEED_R = (MODE != M_L);
    extern __shared__ __align__(128) unsigned char smraw[];
    double* STG = reinterpret_cast<double*>(
        smraw + ((128u - ((unsigned)__cvta_generic_to_shared(smraw) & 127u)) & 127u));
    double* S = STG + T::STG_N;
    double* ACC = S + T::S_N;
    double* FX = ACC + T::ACC_N;
    double* FY = FX + T::FX_N;
    double* CAR = FY + T::FY_N;
    double* sDx = CAR + T::CAR_N;
    double* sDy = sDx + T::DN;
    double* LT = sDy + T::DNY;
    uint64_t* mbarp = reinterpret_cast<uint64_t*>(LT + T::NTAB * a.g.Z);
    uint64_t& mbar = *mbarp;

    const Geo& g = a.g;
    const int Z = g.Z;
    const int tid = threadIdx.x;
    const int ex0 = g.ex_b + blockIdx.x * TX;
    const int ey0 = g.ey_b + blockIdx.y * TY;
    const int nxe = min(TX, g.ex_e - ex0);
    const int nye = min(TY, g.ey_e - ey0);
    const int oxn = nxe * N + ((ex0 + nxe == g.nex) ? 1 : 0);
    const int oyn = nye * NY + ((ey0 + nye == g.ney) ? 1 : 0);
    const int gxlo = (ex0 - 1) * N, gylo = (ey0 - 1) * NY;
    const double gr = a.ph.g;

    if (tid == 0) {
        mbar_init(&mbar, 1);
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
    }
    for (int i = tid; i < T::DN; i += BLK) sDx[i] = a.Dx[i];
    for (int i = tid; i < T::DNY; i += BLK) sDy[i] = a.Dy[i];
    for (int k = tid; k < Z; k += BLK) {
        LT[T_RHO0 * Z + k] = a.lv.rho0[k];
        LT[T_TH0 * Z + k] = a.lv.theta0[k];
        LT[T_E0 * Z + k] = a.lv.E0[k];
        LT[T_C0 * Z + k] = a.lv.c0[k];
        LT[T_IRT0 * Z + k] = a.lv.irt0[k];
        LT[T_G0 * Z + k] = a.lv.G0[k];
        LT[T_H0 * Z + k] = a.lv.H0[k];
        LT[T_DRHO0 * Z + k] = a.lv.drho0[k];
        LT[T_DTH0 * Z + k] = a.lv.dth0[k];
        LT[T_CZ * Z + k] = a.cz[k];
        LT[T_P0F * Z + k] = a.lv.P0f[k];
        LT[T_IRHO0 * Z + k] = 1.0 / a.lv.rho0[k];
    }
    __syncthreads();
    const int txr = gxlo - g.x0, ty0 = gylo - g.y0;
    const int xsh = txr & 1;            // TMA x-origin floored to even (tools/tma_probe.cu)
    const int tx0 = txr - xsh;
    const bool use_tma = a.use_tma != 0;
    if (use_tma) {
        if (tid == 0) {
            mbar_expect_tx(&mbar, T::TMA_BYTES);
            tma_load_4d(STG, &tmap, &mbar, tx0, ty0, 0, 0);
        }
    } else {
        stage_manual3<N, NY, TX, TY>(STG, a, tx0, ty0, 0);
        __syncthreads();
    }

    // main point of this thread (fixed for the sweep): ox fastest
    const int mox = tid % T::OX;
    const int moy = (tid / T::OX) % T::OY;
    const int moz = tid / (T::OX * T::OY);
    const bool main_ok = (tid < T::NMAIN) && mox < nxe * N && moy < nye * NY;
    const int mgx = ex0 * N + mox, mgy = ey0 * NY + moy;
    // A/F of the next layer's main point, fetched one layer ahead
    double Ain[5], Fin[5];
    auto prefetch = [&](int ez) {
        if (!main_ok) return;
        const long long o = loff(g, mgx, mgy, ez * N + moz);
        if (MODE == M_S2) {
#pragma unroll
            for (int f = 0; f < 5; ++f) Ain[f] = a.A[o + f * g.fs];
        }
        if (MODE == M_S2 || MODE == M_S3) {
#pragma unroll
            for (int f = 0; f < 5; ++f) Fin[f] = a.F[o + f * g.fs];
        }
    };
    prefetch(0);

    // per-thread conversion coordinates (levels 1..N of every layer)
    int ccx[T::CONV_IT], ccy[T::CONV_IT], ccz[T::CONV_IT];
#pragma unroll
    for (int it = 0; it < T::CONV_IT; ++it) {
        const int idx = it * BLK + tid;
        ccx[it] = idx % T::LX;
        ccy[it] = (idx / T::LX) % T::LY;
        ccz[it] = 1 + idx / (T::LX * T::LY);
    }
    const double* bc = a.bc;

    for (int ez = 0; ez < g.nez; ++ez) {
        const int base = ez * N;
        const bool last = (ez == g.nez - 1);
        const int ozn = N + (last ? 1 : 0);
        double* CARw = CAR + (ez & 1) * (7 * EY * EX);
        const double* CARr = CAR + ((ez + 1) & 1) * (7 * EY * EX);
        // ------------- C: staged layer -> ring slots -------------------------
        if (use_tma) mbar_wait(&mbar, ez & 1);
        auto convert = [&](int lz, int ly, int lx) {
            const int gz = base + lz;
            const int st = (lz * T::LY + ly) * LXT + lx + xsh;
            const double r = STG[0 * SF + st], u = STG[1 * SF + st], v = STG[2 * SF + st],
                         w = STG[3 * SF + st], th = STG[4 * SF + st];
            double pp = 0.0;
            if (NEED_R)
                pp = pprime(r, th, LT[T_RHO0 * Z + gz], LT[T_TH0 * Z + gz], LT[T_E0 * Z + gz],
                            LT[T_C0 * Z + gz], LT[T_IRT0 * Z + gz], LT[T_P0F * Z + gz], bc, a.ph);
            const int d = ((gz % NL) * T::LY + ly) * LXT + lx;
            S[0 * SF + d] = r;
            S[1 * SF + d] = u;
            S[2 * SF + d] = v;
            S[3 * SF + d] = w;
            S[4 * SF + d] = th;
            S[5 * SF + d] = pp;
        };
        if (ez == 0)
            for (int idx = tid; idx < T::LY * T::LX; idx += BLK) convert(0, idx / T::LX, idx % T::LX);
#pragma unroll
        for (int it = 0; it < T::CONV_IT; ++it)
            if (it * BLK + tid < T::CONV_N) convert(ccz[it], ccy[it], ccx[it]);
        __syncthreads();
        if (use_tma) {
            if (tid == 0 && ez + 1 < g.nez) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(&mbar, T::TMA_BYTES);
                tma_load_4d(STG, &tmap, &mbar, tx0, ty0, base + N, 0);
            }
        } else if (ez + 1 < g.nez) {
            stage_manual3<N, NY, TX, TY>(STG, a, tx0, ty0, base + N);
        }

        // ------------- X: element x-lines ------------------------------------
        if (NEED_R) {
            constexpr int NXI = 2 * (TX + 1) * EY * NZL;
            for (int it = tid; it < NXI; it += BLK) {
                const int grp = it & 1;
                int t = it >> 1;
                const int ae = t % (TX + 1);
                t /= (TX + 1);
                const int oy = t % EY;
                const int oz = t / EY;
                const int xe = ae - 1;
                if (oz >= ozn || oy >= oyn || xe >= nxe) continue;
                if (xe < 0 && ex0 == 0) continue;               // no element left of the domain
                const int fox = (xe + 1) * N;                    // the line's row-N point
                const bool face_own = fox < oxn;                 // is it owned by this tile?
                if (xe < 0 && !face_own) continue;
                const int gz = base + oz;
                const int row = (gz % NL) * PL + (oy + NY) * LXT + ae * N;   // line start
                const double rho0 = LT[T_RHO0 * Z + gz];
                // u and rho at the N+1 line positions
                double ul[N + 1], rl[N + 1];
#pragma unroll
                for (int m = 0; m <= N; ++m) {
                    ul[m] = S[1 * SF + row + m];
                    rl[m] = rho0 + S[0 * SF + row + m];
                }
                // fields of the group: g0 {rho', u, P'} -> ACC0, ACC1; g1 {v, w, theta'} -> ACC2..4
                const int f0 = grp ? 2 : 0, f1 = grp ? 3 : 1, f2 = grp ? 4 : 5;
                double l0[N + 1], l1[N + 1], l2[N + 1];
#pragma unroll
                for (int m = 0; m <= N; ++m) {
                    l0[m] = S[f0 * SF + row + m];
                    l1[m] = S[f1 * SF + row + m];
                    l2[m] = S[f2 * SF + row + m];
                }
                const bool tgt_end = face_own && (ex0 * N + fox == g.X - 1);
#pragma unroll
                for (int i = 0; i <= N; ++i) {
                    if (i < N && xe < 0) continue;               // halo element: row N only
                    if (i == N && !face_own) continue;
                    double d0 = 0.0, d1 = 0.0, d2 = 0.0;
#pragma unroll
                    for (int m = 0; m <= N; ++m) {
                        const double dm = sDx[i * (N + 1) + m];
                        d0 = fma(dm, l0[m], d0);
                        d1 = fma(dm, l1[m], d1);
                        d2 = fma(dm, l2[m], d2);
                    }
                    const int ox = xe * N + i;                   // == fox for i == N
                    const double c = __ldg(a.cx + ex0 * N + ox);
                    const double u = ul[i], rho = rl[i];
                    double c0, c1, c2 = 0.0;
                    if (grp == 0) {          // u d(rho') + rho d(u) ;  u d(u) + d(P')/rho
                        c0 = c * (u * d0 + rho * d1);
                        c1 = c * (u * d1 + d2 / rho);
                    } else {                 // u d(v) ; u d(w) ; u d(theta')
                        c0 = c * (u * d0);
                        c1 = c * (u * d1);
                        c2 = c * (u * d2);
                    }
                    const int p = (oz * EY + oy) * EX + ox;
                    if (i < N || tgt_end) {                      // own (or the domain end)
                        if (grp == 0) {
                            ACC[0 * NPT + p] = c0;
                            ACC[1 * NPT + p] = c1;
                        } else {
                            ACC[2 * NPT + p] = c0;
                            ACC[3 * NPT + p] = c1;
                            ACC[4 * NPT + p] = c2;
                        }
                    } else {                                     // face partial from the left
                        const int q = (oz * EY + oy) * (TX + 1) + (ae);
                        constexpr int FS = NZL * EY * (TX + 1);
                        if (grp == 0) {
                            FX[0 * FS + q] = c0;
                            FX[1 * FS + q] = c1;
                        } else {
                            FX[2 * FS + q] = c0;
                            FX[3 * FS + q] = c1;
                            FX[4 * FS + q] = c2;
                        }
                    }
                }
            }
        }
        __syncthreads();
        // ------------- Y: element y-lines ------------------------------------
        if (NEED_R) {
            constexpr int NYI = 2 * (TY + 1) * EX * NZL;
            for (int it = tid; it < NYI; it += BLK) {
                const int grp = it & 1;
                int t = it >> 1;
                const int ox = t % EX;
                t /= EX;
                const int be = t % (TY + 1);
                const int oz = t / (TY + 1);
                const int ye = be - 1;
                if (oz >= ozn || ox >= oxn || ye >= nye) continue;
                if (ye < 0 && ey0 == 0) continue;
                const int foy = (ye + 1) * NY;
                const bool face_own = foy < oyn;
                if (ye < 0 && !face_own) continue;
                const int gz = base + oz;
                const int col = (gz % NL) * PL + (be * NY) * LXT + ox + N;   // line start (m = 0)
                const double rho0 = LT[T_RHO0 * Z + gz];
                double vl[NY + 1], rl[NY + 1];
#pragma unroll
                for (int m = 0; m <= NY; ++m) {
                    vl[m] = S[2 * SF + col + m * LXT];
                    rl[m] = rho0 + S[0 * SF + col + m * LXT];
                }
                // g0 {rho', v, P'} -> ACC0, ACC2 ; g1 {u, w, theta'} -> ACC1, ACC3, ACC4
                const int f0 = grp ? 1 : 0, f1 = grp ? 3 : 2, f2 = grp ? 4 : 5;
                double l0[NY + 1], l1[NY + 1], l2[NY + 1];
#pragma unroll
                for (int m = 0; m <= NY; ++m) {
                    l0[m] = S[f0 * SF + col + m * LXT];
                    l1[m] = S[f1 * SF + col + m * LXT];
                    l2[m] = S[f2 * SF + col + m * LXT];
                }
                const bool tgt_end = face_own && (ey0 * NY + foy == g.Y - 1);
#pragma unroll
                for (int j = 0; j <= NY; ++j) {
                    if (j < NY && ye < 0) continue;
                    if (j == NY && !face_own) continue;
                    double d0 = 0.0, d1 = 0.0, d2 = 0.0;
#pragma unroll
                    for (int m = 0; m <= NY; ++m) {
                        const double dm = sDy[j * (NY + 1) + m];
                        d0 = fma(dm, l0[m], d0);
                        d1 = fma(dm, l1[m], d1);
                        d2 = fma(dm, l2[m], d2);
                    }
                    const int oy = ye * NY + j;
                    const double c = __ldg(a.cy + ey0 * NY + oy);
                    const double v = vl[j], rho = rl[j];
                    double c0, c1, c2 = 0.0;
                    if (grp == 0) {          // v d(rho') + rho d(v) ;  v d(v) + d(P')/rho
                        c0 = c * (v * d0 + rho * d1);
                        c1 = c * (v * d1 + d2 / rho);
                    } else {                 // v d(u) ; v d(w) ; v d(theta')
                        c0 = c * (v * d0);
                        c1 = c * (v * d1);
                        c2 = c * (v * d2);
                    }
                    const int p = (oz * EY + oy) * EX + ox;
                    if (j < NY || tgt_end) {
                        if (grp == 0) {
                            ACC[0 * NPT + p] += c0;
                            ACC[2 * NPT + p] += c1;
                        } else {
                            ACC[1 * NPT + p] += c0;
                            ACC[3 * NPT + p] += c1;
                            ACC[4 * NPT + p] += c2;
                        }
                    } else {
                        const int q = (oz * EX + ox) * (TY + 1) + be;
                        constexpr int FS = NZL * EX * (TY + 1);
                        if (grp == 0) {
                            FY[0 * FS + q] = c0;
                            FY[2 * FS + q] = c1;
                        } else {
                            FY[1 * FS + q] = c0;
                            FY[3 * FS + q] = c1;
                            FY[4 * FS + q] = c2;
                        }
                    }
                }
            }
        }
        __syncthreads();
        // ------------- Z: the layer's z-line of every owned column -----------
        {
            constexpr int NZI = 3 * EX * EY;
            int zsl[N + 1];
#pragma unroll
            for (int m = 0; m <= N; ++m) zsl[m] = ((base + m) % NL) * PL;
            for (int it = tid; it < NZI; it += BLK) {
                const int grp = it % 3;
                const int c = it / 3;
                const int ox = c % EX, oy = c / EX;
                if (ox >= oxn || oy >= oyn) continue;
                if (!NEED_R && grp == 1) continue;
                const int cidx = oy * EX + ox;
                const int col = (oy + NY) * LXT + ox + N;
                double wl[N + 1], l0[N + 1], l1[N + 1], l2[N + 1];
                int fa, fb, fc;   // carry slots of the three lines
#pragma unroll
                for (int m = 0; m <= N; ++m) wl[m] = S[3 * SF + zsl[m] + col];
                if (grp == 0) {          // rho', w, P'  -> ACC0, ACC3, ACC5(L0)
                    fa = 0; fb = 3; fc = 5;
#pragma unroll
                    for (int m = 0; m <= N; ++m) {
                        l0[m] = S[0 * SF + zsl[m] + col];
                        l1[m] = wl[m];
                        l2[m] = NEED_R ? S[5 * SF + zsl[m] + col] : 0.0;
                    }
                } else if (grp == 1) {   // u, v -> ACC1, ACC2
                    fa = 1; fb = 2; fc = -1;
#pragma unroll
                    for (int m = 0; m <= N; ++m) {
                        l0[m] = S[1 * SF + zsl[m] + col];
                        l1[m] = S[2 * SF + zsl[m] + col];
                        l2[m] = 0.0;
                    }
                } else {                 // theta', Plin -> ACC4, ACC6(L3)
                    fa = 4; fb = 6; fc = -1;
#pragma unroll
                    for (int m = 0; m <= N; ++m) {
                        const int gzm = base + m;
                        const double rr = S[0 * SF + zsl[m] + col], tt = S[4 * SF + zsl[m] + col];
                        l0[m] = tt;
                        l1[m] = NEED_L ? LT[T_G0 * Z + gzm] * rr + LT[T_H0 * Z + gzm] * tt : 0.0;
                        l2[m] = 0.0;
                    }
                }
                // carry (row N) into the next layer
                if (ez + 1 < g.nez) {
                    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
                    for (int m = 0; m <= N; ++m) {
                        const double dm = sDx[N * (N + 1) + m];
                        s0 = fma(dm, l0[m], s0);
                        s1 = fma(dm, l1[m], s1);
                        s2 = fma(dm, l2[m], s2);
                    }
                    CARw[fa * (EY * EX) + cidx] = s0;
                    CARw[fb * (EY * EX) + cidx] = s1;
                    if (fc >= 0) CARw[fc * (EY * EX) + cidx] = s2;
                }
#pragma unroll
                for (int k = 0; k <= N; ++k) {
                    if (k == N && !last) continue;
                    const int gz = base + k;
                    double d0 = 0.0, d1 = 0.0, d2 = 0.0;
#pragma unroll
                    for (int m = 0; m <= N; ++m) {
                        const double dm = sDx[k * (N + 1) + m];
                        d0 = fma(dm, l0[m], d0);
                        d1 = fma(dm, l1[m], d1);
                        d2 = fma(dm, l2[m], d2);
                    }
                    if (k == 0 && ez > 0) {
                        d0 += CARr[fa * (EY * EX) + cidx];
                        d1 += CARr[fb * (EY * EX) + cidx];
                        if (fc >= 0) d2 += CARr[fc * (EY * EX) + cidx];
                    }
                    const double cz = LT[T_CZ * Z + gz];
                    const double w = wl[k];
                    const int p = (k * EY + oy) * EX + ox;
                    if (grp == 0) {
                        const double rho0 = LT[T_RHO0 * Z + gz];
                        if (NEED_R) {
                            const double rho = rho0 + l0[k];
                            ACC[0 * NPT + p] += cz * (w * d0 + rho * d1);   // w d(rho') + rho d(w)
                            ACC[3 * NPT + p] += cz * (w * d1 + d2 / rho);   // w d(w) + d(P')/rho
                        }
                        if (NEED_L) ACC[5 * NPT + p] = rho0 * (cz * d1);    // rho0 d(w)/dz
                    } else if (grp == 1) {
                        ACC[1 * NPT + p] += cz * (w * d0);                  // w d(u)
                        ACC[2 * NPT + p] += cz * (w * d1);                  // w d(v)
                    } else {
                        if (NEED_R) ACC[4 * NPT + p] += cz * (w * d0);      // w d(theta')
                        if (NEED_L) ACC[6 * NPT + p] = cz * d1;             // d(Plin)/dz
                    }
                }
            }
        }
        __syncthreads();
        // ------------- F: pointwise terms + ARK2 epilogue ---------------------
        auto finish = [&](int ox, int oy, int oz, const double* Ai, const double* Fi) {
            const int gx = ex0 * N + ox, gy = ey0 * NY + oy, gz = base + oz;
            const int p = (oz * EY + oy) * EX + ox;
            const int pnt = (gz % NL) * PL + (oy + NY) * LXT + ox + N;
            const double r = S[0 * SF + pnt], u = S[1 * SF + pnt], v = S[2 * SF + pnt],
                         w = S[3 * SF + pnt], th = S[4 * SF + pnt];
            const double rho0 = LT[T_RHO0 * Z + gz];
            const double drho0 = LT[T_DRHO0 * Z + gz];
            const double dth0 = LT[T_DTH0 * Z + gz];
            const bool bx = (gx == 0) || (gx == g.X - 1);
            const bool by = g.slab || (gy == 0) || (gy == g.Y - 1);
            const bool bz = (gz == 0) || (gz == g.Z - 1);
            double Rv[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
            if (NEED_R) {
                const double rho = rho0 + r;
                const double theta = LT[T_TH0 * Z + gz] + th;
                if (!(isfinite(r) && isfinite(u) && isfinite(v) && isfinite(w) && isfinite(th)))
                    atomicOr(a.flags, HEVI_F_NONFINITE_IN(a.stage));
                if (!(rho > 0.0) || !(theta > 0.0)) atomicOr(a.flags, HEVI_F_EOS(a.stage));
                double acc[5];
#pragma unroll
                for (int c = 0; c < 5; ++c) acc[c] = ACC[c * NPT + p];
                const bool xf = (ox % N == 0) && gx > 0 && gx < g.X - 1;
                const bool yf = (oy % NY == 0) && gy > 0 && gy < g.Y - 1;
                if (xf) {
                    constexpr int FS = NZL * EY * (TX + 1);
                    const int q = (oz * EY + oy) * (TX + 1) + ox / N;
#pragma unroll
                    for (int c = 0; c < 5; ++c) acc[c] += FX[c * FS + q];
                }
                if (yf) {
                    constexpr int FS = NZL * EX * (TY + 1);
                    const int q = (oz * EX + ox) * (TY + 1) + oy / NY;
#pragma unroll
                    for (int c = 0; c < 5; ++c) acc[c] += FY[c * FS + q];
                }
                // euler.nonlinear_rhs set2nc (euler.py:458-473) with the DSS folded into the
                // derivatives; no-flux projection after the DSS (euler.py:494-496)
                Rv[0] = -(acc[0] + w * drho0);
                Rv[1] = bx ? 0.0 : -acc[1];
                Rv[2] = by ? 0.0 : -acc[2];
                Rv[3] = bz ? 0.0 : -(acc[3] + (r / rho) * gr);
                Rv[4] = -(acc[4] + w * dth0);
            }
            double Lv[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
            if (NEED_L) {
                // euler.linear_operator(vertical_only=True), set2nc (euler.py:333-361)
                const double irho0 = LT[T_IRHO0 * Z + gz];
                Lv[0] = -(w * drho0 + ACC[5 * NPT + p]);
                Lv[3] = bz ? 0.0 : -(ACC[6 * NPT + p] * irho0 + (r * irho0) * gr);
                Lv[4] = -(w * dth0);
            }
            const long long o = loff(g, gx, gy, gz);
            const long long fs = g.fs;
            if (MODE == M_R) {
#pragma unroll
                for (int f = 0; f < 5; ++f) a.out[o + f * fs] = Rv[f];
            } else if (MODE == M_L) {
#pragma unroll
                for (int f = 0; f < 5; ++f) a.out[o + f * fs] = Lv[f];
            } else if (MODE == M_S1) {
                // imexcore.ark_imex_step (imexcore.py:398-403, 409-411)
                const double dt = a.dt;
                const double qv[5] = {r, u, v, w, th};
                double pr[5];
#pragma unroll
                for (int f = 0; f < 5; ++f) {
                    pr[f] = qv[f] + dt * (a.a_p * (Rv[f] - Lv[f]) + a.at_p * Lv[f]);
                    a.A[o + f * fs] = qv[f] + dt * (a.a_a * (Rv[f] - Lv[f]) + a.at_a * Lv[f]);
                    a.F[o + f * fs] = qv[f] + a.cb * Rv[f];
                }
                a.P[o] = pr[0];
                a.P[o + 3 * fs] = pr[3];
                a.P[o + 4 * fs] = pr[4];
                a.Quv[o + fs] = bx ? 0.0 : pr[1];
                a.Quv[o + 2 * fs] = by ? 0.0 : pr[2];
            } else if (MODE == M_S2) {
                const double dt = a.dt;
                double pr[5];
#pragma unroll
                for (int f = 0; f < 5; ++f) {
                    pr[f] = Ai[f] + dt * (a.a_p * (Rv[f] - Lv[f]) + a.at_p * Lv[f]);
                    a.F[o + f * fs] = Fi[f] + a.cb * Rv[f];
                }
                a.P[o] = pr[0];
                a.P[o + 3 * fs] = pr[3];
                a.P[o + 4 * fs] = pr[4];
                a.Quv[o + fs] = bx ? 0.0 : pr[1];
                a.Quv[o + 2 * fs] = by ? 0.0 : pr[2];
            } else {
                bool fin = true;
#pragma unroll
                for (int f = 0; f < 5; ++f) {
                    const double val = Fi[f] + a.cb * Rv[f];
                    fin = fin && isfinite(val);
                    a.out[o + f * fs] = val;
                }
                if (!fin) atomicOr(a.flags, HEVI_F_NONFINITE_OUT);
            }
        };
        if (main_ok) finish(mox, moy, moz, Ain, Fin);
        if (ez + 1 < g.nez) prefetch(ez + 1);
        // points outside the main box: domain-end column/row, top level
        const int mainx = nxe * N, mainy = nye * NY;
        const int nfull = oxn * oyn * ozn;
        if (nfull > mainx * mainy * N) {
            for (int p = tid; p < nfull; p += BLK) {
                const int ox = p % oxn;
                const int t = p / oxn;
                const int oy = t % oyn;
                const int oz = t / oyn;
                if (ox < mainx && oy < mainy && oz < N) continue;
                double Ae[5], Fe[5];
                const long long o = loff(g, ex0 * N + ox, ey0 * NY + oy, base + oz);
#pragma unroll
                for (int f = 0; f < 5; ++f) {
                    Ae[f] = (MODE == M_S2) ? a.A[o + f * g.fs] : 0.0;
                    Fe[f] = (MODE == M_S2 || MODE == M_S3) ? a.F[o + f * g.fs] : 0.0;
                }
                finish(ox, oy, oz, Ae, Fe);
            }
        }
        __syncthreads();
    }
}
