// explicit_col.cuh -- column-sweep explicit kernel for 3D boxes, N = 4
// (included by hevi.cu inside its anonymous namespace, after explicit_v2.cuh).
//
// R(q) (euler.nonlinear_rhs set2nc, euler.py:438-497), L_V(q)
// (euler.vertical_restriction, euler.py:313-371) and the fused ARK2 stage
// epilogues (imexcore.ark_imex_step, imexcore.py:385-414), with the DSS
// folded into the derivatives exactly as k_explicit2 does.
//
// Structure (one CTA per 4x4-element horizontal tile, one thread per owned
// lattice column, 256 threads, sweeping the levels bottom-up):
//   * every level of the tile (+ N halo points low side, 1 high side) arrives
//     by TMA into a ring of S level slots (6 planes: rho', u, v, w, theta',
//     P'); a slot is refilled S levels ahead as soon as its level is done;
//   * the z-lines never touch shared memory after the window load: at each
//     element layer a thread loads its column's N+1 levels of the 6 fields
//     into a register window, and every vertical derivative of the layer is
//     a register contraction with the D row of the level (uniform loads from
//     the parameter bank); the element-face carry from the layer below is a
//     register too;
//   * x-lines are element lines starting on 32-byte boundaries: two 16-byte
//     and one 8-byte shared load per field; the row pitch (22 doubles) makes
//     the warp's 2 rows x 4 elements conflict-free; y-lines are broadcast
//     across the warp's two rows (one wavefront per load);
//   * element-face partial sums (row N of the left / lower element) of the
//     next level are formed once per face by all threads and double-buffered
//     across the per-level barrier;
//   * the domain-end planes x = X-1 and y = Y-1 (0.3% of the points) are
//     evaluated by k_ecol_edge, one thread per point, lines from global.
// Per-level constants (reference state, metric factor cz, the D rows of the
// vertical derivative, the EOS reference point) sit in a __grid_constant__
// parameter block: warp-uniform indices, no shared-memory bandwidth.
#pragma once

#define EC_ZMAX 64
// domain-end kernel as a programmatic dependent launch of the sweep (else
// forked onto the plan's side stream): measured per equation set -- set2c
// 4.35 -> 4.15 ms per step with it; set2nc within 0.3 % at one GPU and 1-2 %
// slower at the x-end ranks of 2/4/8-GPU windows, so set2nc forks
#ifndef HEVI_EDGE_PDL_NC
#define HEVI_EDGE_PDL_NC 0
#endif
#ifndef HEVI_EDGE_PDL_C
#define HEVI_EDGE_PDL_C 1
#endif
#define EC_NMAX 4
#ifndef HEVI_ECOL_TY
#define HEVI_ECOL_TY 4   // tile rows in elements (2: two 128-thread CTAs per SM)
#endif
enum { C_RHO0 = 0, C_TH0, C_DRHO0, C_DTH0, C_CZ, C_IRHO0, C_G0, C_H0, C_PB, C_C0, C_IRT0, C_P0F,
       C_TH0C, C_ITH0, C_F0C, EC_NT };   // set2c: Theta0 = rho0 theta0, 1/Theta0, F0 = gamma P0f / Theta0

// per-level constants of the explicit_col kernels (N <= EC_NMAX, Z <= EC_ZMAX);
// row(l) = l mod N (N on the top level), base(l) = l - row(l)
struct LvlTab {
    double v[EC_NT][EC_ZMAX];
    double dx[25], dy[25], dz[25];   // (N+1)^2 derivative matrices, row-major
    double dzs[EC_ZMAX][5];          // cz[l] * Dz[row(l)][m]: the level's scaled vertical D row
    double czf[EC_ZMAX];             // cz[l] on a bottom element face (carry from below), else 0
    double pg[EC_ZMAX][5], ph[EC_ZMAX][5];   // dzs[l][m] * G0 / H0 [base(l) + m]: d/dz of P_lin
    double cg[EC_ZMAX][5], ch[EC_ZMAX][5];   // Dz[N][m] * G0 / H0 [l + m]: row-N carry of P_lin, layer base l
};

// the tile of this CTA (EArgs::tmode): the whole grid, the interior
// rectangle, or the i-th tile of the ring around it (bottom rows, top rows,
// then the left / right tiles of the middle rows)
__device__ __forceinline__ void ec_tile(const EArgs& a, int& bx, int& by) {
    if (a.tmode == 0) {
        bx = blockIdx.x;
        by = blockIdx.y;
    } else if (a.tmode == 1) {
        bx = a.tb[2] + blockIdx.x;
        by = a.tb[4] + blockIdx.y;
    } else {
        const int nbx = a.tb[0], nby = a.tb[1], bx0 = a.tb[2], bx1 = a.tb[3], by0 = a.tb[4], by1 = a.tb[5];
        int i = blockIdx.x;
        const int nlow = by0 * nbx, nhigh = (nby - by1) * nbx;
        if (i < nlow) {
            by = i / nbx;
            bx = i % nbx;
        } else if ((i -= nlow) < nhigh) {
            by = by1 + i / nbx;
            bx = i % nbx;
        } else {
            i -= nhigh;
            const int wl = bx0, w = bx0 + (nbx - bx1);
            by = by0 + i / w;
            const int r = i % w;
            bx = r < wl ? r : bx1 + (r - wl);
        }
    }
}

// TMA bulk tensor store of one staged box (shared::cta -> global)
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* src, int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(map),
        "r"((unsigned)__cvta_generic_to_shared(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

template <int K>
struct KI {
    static constexpr int v = K;
};

template <int N, int MODE>
struct EC {
    static constexpr int TX = 4, TY = HEVI_ECOL_TY;           // elements per tile
    static constexpr int OX = TX * N, OY = TY * N;            // owned columns
    static constexpr int BLK = OX * OY;                       // one thread per column
    static constexpr int LX = OX + N + 1, LY = OY + N + 1;    // staged extent
    static constexpr int LXT = (LX + 1) / 2 * 2;              // TMA box x (16-byte multiple)
    static constexpr int PL = LXT * LY;                       // one field plane
    static constexpr int PPO = (5 * PL + 15) / 16 * 16;       // P' plane (128-byte aligned)
    static constexpr int SS = (PPO + PL + 15) / 16 * 16;      // slot stride
    // pointwise stage inputs (A and/or F) of a level: TMA boxes OX x OY x 5
    static constexpr int NAF = (MODE == M_S2) ? 2 : (MODE == M_S3) ? 1 : 0;
    static constexpr int SAF = NAF ? 2 : 0;                   // A/F level slots
    static constexpr int SAFM = NAF ? SAF : 1;                // (modulus when SAF is 0)
    static constexpr int AFB = 5 * OX * OY;                   // one array's box
    // stage 0's A and F outputs (10 planes) leave by TMA bulk tensor stores
    // from a double-buffered staging area: no per-store address arithmetic.
    // (Staging every output of every stage measured slower: 3.48 vs 3.27 ms.)
    static constexpr int NOUT = (MODE == M_S1) ? 10 : 0;
    static constexpr int S = NAF ? 6 : (NOUT ? (TY == 4 ? 7 : 6) : 8);   // ring slots
    static constexpr int NXF = 6 * OY * TX, NYF = 6 * TY * OX;   // face partials per level
    static constexpr int DN = (N + 1) * (N + 1);
    static constexpr size_t SMEM =
        sizeof(double) * ((size_t)S * SS + (size_t)SAF * NAF * AFB + 2 * (size_t)NOUT * OX * OY +
                          2 * (NXF + NYF) + 2 * DN + OX + OY) +
        sizeof(uint64_t) * (S + SAF) + 128;
    static constexpr uint32_t LVL_BYTES = (uint32_t)(sizeof(double) * 5 * PL);
    static constexpr uint32_t PP_BYTES = (uint32_t)(sizeof(double) * PL);
    static constexpr uint32_t AF_BYTES = (uint32_t)(sizeof(double) * AFB);
    __host__ __device__ static constexpr int foff(int f) { return f < 5 ? f * PL : PPO; }
};

// R(q), L_V(q) at one point, accumulated field by field from its derivative
// values (euler.py:458-473, 333-361); the no-flux projection
// (euler.py:494-496) on the domain faces
struct PtSt {
    double r, u, v, w, th, rho, rinv;
};
struct PtAcc {
    double R0, R1, R2, R3, R4, divu, dwz, dPLz;
};

__device__ __forceinline__ void ec_fold(int f, double gx, double gy, double gz, const PtSt& p, PtAcc& c) {
    switch (f) {
        case 0: c.R0 = (p.u * gx + p.v * gy) + p.w * gz; break;
        case 1: c.R1 = (p.u * gx + p.v * gy) + p.w * gz; c.divu = gx; break;
        case 2: c.R2 = (p.u * gx + p.v * gy) + p.w * gz; c.divu += gy; break;
        case 3: c.R3 = (p.u * gx + p.v * gy) + p.w * gz; c.divu += gz; c.dwz = gz; break;
        case 4: c.R4 = (p.u * gx + p.v * gy) + p.w * gz; break;
        case 5:
            c.R1 += gx * p.rinv;
            c.R2 += gy * p.rinv;
            c.R3 += gz * p.rinv;
            c.R0 += p.rho * c.divu;
            break;
        default: c.dPLz = gz; break;
    }
}

template <int MODE>
__device__ __forceinline__ void ec_finish(const PtSt& p, const PtAcc& c, double rho0, double drho0,
                                          double dth0, double irho0, double gr, bool bx, bool by, bool bz,
                                          double (&Rv)[5], double (&Lv)[5]) {
    constexpr bool NEED_L = (MODE == M_L || MODE == M_S1 || MODE == M_S2);
    constexpr bool NEED_R = (MODE != M_L);
#pragma unroll
    for (int f = 0; f < 5; ++f) Rv[f] = Lv[f] = 0.0;
    if (NEED_R) {
        Rv[0] = -(c.R0 + p.w * drho0);
        Rv[1] = bx ? 0.0 : -c.R1;
        Rv[2] = by ? 0.0 : -c.R2;
        Rv[3] = bz ? 0.0 : -(c.R3 + (p.r * p.rinv) * gr);
        Rv[4] = -(c.R4 + p.w * dth0);
    }
    if (NEED_L) {
        Lv[0] = -(p.w * drho0 + rho0 * c.dwz);
        Lv[3] = bz ? 0.0 : -(c.dPLz * irho0 + (p.r * irho0) * gr);
        Lv[4] = -(p.w * dth0);
    }
}

// input checks of nonlinear_rhs (euler.py:445-446, 183-184) at one point
__device__ __forceinline__ void ec_check(const EArgs& a, const PtSt& p, double th0) {
    const double s = ((p.r + p.u) + (p.v + p.w)) + p.th;
    if (!isfinite(s)) {
        if (!(isfinite(p.r) && isfinite(p.u) && isfinite(p.v) && isfinite(p.w) && isfinite(p.th)))
            atomicOr(a.flags, HEVI_F_NONFINITE_IN(a.stage));
    }
    if (!(p.rho > 0.0) || !(th0 + p.th > 0.0)) atomicOr(a.flags, HEVI_F_EOS(a.stage));
}

// the same checks as flag bits, branch-free (accumulated over the sweep, one
// atomic per thread at the end): x * 0 is NaN exactly for a non-finite x
__device__ __forceinline__ unsigned ec_bits(const EArgs& a, const PtSt& p, double th0) {
    const double z = fma(p.r, 0.0, fma(p.u, 0.0, fma(p.v, 0.0, fma(p.w, 0.0, p.th * 0.0))));
    unsigned b = (z == z) ? 0u : HEVI_F_NONFINITE_IN(a.stage);
    b |= (p.rho > 0.0 && th0 + p.th > 0.0) ? 0u : HEVI_F_EOS(a.stage);
    return b;
}

// P' of a point from the per-level EOS constants (pprime of explicit_v2.cuh)
__device__ __forceinline__ double ec_pprime(const EArgs& a, const LvlTab& lt, int gz, double r,
                                            double th) {
    return pprime(r, th, lt.v[C_RHO0][gz], lt.v[C_TH0][gz], lt.v[C_PB][gz], lt.v[C_C0][gz],
                  lt.v[C_IRT0][gz], lt.v[C_P0F][gz], a.bc, a.ph);
}

// fused ARK2 stage epilogues (imexcore.py:398-411) and the plain R / L outputs
template <int MODE>
__device__ __forceinline__ void ec_epilogue(const EArgs& a, const LvlTab& lt, long long o, int gz,
                                            const PtSt& p, const double (&Rv)[5], const double (&Lv)[5],
                                            const double (&Ai)[5], const double (&Fi)[5], bool bx,
                                            bool by, bool own = true, unsigned* fl = nullptr) {
    const long long fs = a.g.fs;
    if (!own) return;
    if (MODE == M_R) {
#pragma unroll
        for (int f = 0; f < 5; ++f) a.out[o + f * fs] = Rv[f];
    } else if (MODE == M_L) {
#pragma unroll
        for (int f = 0; f < 5; ++f) a.out[o + f * fs] = Lv[f];
    } else if (MODE == M_S1) {
        const double dt = a.dt;
        const double qv[5] = {p.r, p.u, p.v, p.w, p.th};
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
    } else if (MODE == M_S3) {
        double qn[5];
        bool fin = true;
#pragma unroll
        for (int f = 0; f < 5; ++f) {
            qn[f] = Fi[f] + a.cb * Rv[f];
            fin = fin && isfinite(qn[f]);
            a.out[o + f * fs] = qn[f];
        }
        if (fl) *fl |= fin ? 0u : HEVI_F_NONFINITE_OUT;
        else if (!fin) atomicOr(a.flags, HEVI_F_NONFINITE_OUT);
        // P' of the new state for the next step's stage 0 (replaces k_pp_plane)
        if (a.pp_out && fin) a.pp_out[o] = ec_pprime(a, lt, gz, qn[0], qn[4]);
    }
}

template <int N, int MODE>
__global__ void __launch_bounds__(EC<N, MODE>::BLK, 4 / HEVI_ECOL_TY)
    k_ecol(const EArgs a, const __grid_constant__ LvlTab lt, const __grid_constant__ CUtensorMap tmq,
           const __grid_constant__ CUtensorMap tmp, const __grid_constant__ CUtensorMap tmA,
           const __grid_constant__ CUtensorMap tmF, const __grid_constant__ CUtensorMap tmO0,
           const __grid_constant__ CUtensorMap tmO1, const __grid_constant__ CUtensorMap tmO2,
           const __grid_constant__ CUtensorMap tmO3) {
    using T = EC<N, MODE>;
    constexpr int LXT = T::LXT, SS = T::SS, S = T::S, BLK = T::BLK;
    constexpr int OX = T::OX, OY = T::OY, TX = T::TX, TY = T::TY;
    constexpr bool NEED_L = (MODE == M_L || MODE == M_S1 || MODE == M_S2);
    constexpr bool NEED_R = (MODE != M_L);
    static_assert(N == 4, "x-line vector loads assume N = 4");
    extern __shared__ __align__(128) unsigned char smraw[];
    double* ring = reinterpret_cast<double*>(
        smraw + ((128u - ((unsigned)__cvta_generic_to_shared(smraw) & 127u)) & 127u));
    double* sAF = ring + S * SS;          // [SAF][NAF][5][OY][OX]: A (M_S2) | F
    double* sOut = sAF + T::SAF * T::NAF * T::AFB;  // [2][NOUT][OY][OX] staged outputs (TMA store sources)
    double* XFb = sOut + 2 * T::NOUT * OX * OY;     // [2][NXF]  XF[f][oy][j]
    double* YFb = XFb + 2 * T::NXF;       // [2][NYF]  YF[f][j][ox]
    double* sD = YFb + 2 * T::NYF;        // Dx | Dy
    double* sC = sD + 2 * T::DN;          // cx of the tile's columns | cy of its rows
    uint64_t* mbar = reinterpret_cast<uint64_t*>(sC + OX + OY);   // [S] ring, [SAF] A/F

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

    // the domain-end kernel launched after this one (programmatic dependent
    // launch) may start once every tile of this grid is resident: it then
    // fills the SMs the last wave leaves idle instead of delaying that wave
    if (HEVI_EDGE_PDL_NC) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#ifdef HEVI_EDGE_TIMING
    if (tid == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        atomicMax(a.dbg + 0, ~0ull - t);
        atomicMax(a.dbg + 1, t);
    }
#endif
    if (tid == 0) {
        for (int s = 0; s < S + T::SAF; ++s) mbar_init(&mbar[s], 1);
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmq) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmp) : "memory");
    }
    for (int i = tid; i < T::DN; i += BLK) {
        sD[i] = a.Dx[i];
        sD[T::DN + i] = a.Dy[i];
    }
    // metric factors through shared memory: a register loaded from global
    // before the sweep would share a scoreboard with the per-level loads
    if (tid < OX) sC[tid] = (ex0 * N + tid < g.X) ? a.cx[ex0 * N + tid] : 0.0;
    else if (tid < OX + OY) sC[tid] = (ey0 * N + tid - OX < g.Y) ? a.cy[ey0 * N + tid - OX] : 0.0;
    __syncthreads();
    auto issue = [&](int l) {
        double* slot = ring + (l % S) * SS;
        uint64_t* bar = &mbar[l % S];
        mbar_expect_tx(bar, T::LVL_BYTES + T::PP_BYTES);
        tma_load_4d(slot, &tmq, bar, tx0, ty0, l, 0);
        tma_load_4d(slot + T::PPO, &tmp, bar, tx0, ty0, l, 0);
    };
    // A/F boxes of a level (window-local origin of the owned tile)
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

    // per-thread constants
    const int rx = ox % N, ry = oy % N;
    // the thread's D rows scaled by its metric factors (and the face-partial weights)
    const double cxv = own ? sC[ox] : 0.0, cyv = own ? sC[OX + oy] : 0.0;
    double Dxr[N + 1], Dyr[N + 1];
#pragma unroll
    for (int m = 0; m <= N; ++m) {
        Dxr[m] = cxv * sD[rx * (N + 1) + m];
        Dyr[m] = cyv * sD[T::DN + ry * (N + 1) + m];
    }
    // element-face weights; the domain's low walls (gx = 0, gy = 0) have no lower element
    const double fxs = (rx == 0 && gx > 0) ? cxv : 0.0, fys = (ry == 0 && gy > 0) ? cyv : 0.0;
    const bool bx = (gx == 0), by = (gy == 0);   // x = X-1 / y = Y-1: k_ecol_edge
    const int lx = ox + N, ly = oy + N;
    const int xo = ly * LXT + (lx - rx);   // x-line start (32-byte aligned)
    const int yo = (ly - ry) * LXT + lx;   // y-line start
    const int po = ly * LXT + lx;          // own point
    const int xfo = oy * TX + ox / N;
    const int yfo = (oy / N) * OX + ox;
    const long long colo = (long long)(gy - g.y0) * g.px + (gx - g.x0);
    const long long zs = (long long)g.lY * g.px;
    const double gr = a.ph.g;

    // element-face partials (row N of the left / lower element) of level l;
    // a thread's items and their slot offsets are the same on every level
    static_assert(T::NXF + T::NYF <= 3 * BLK, "faces: three items per thread");
    int fo[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        const int i = tid + r * BLK;
        if (i < T::NXF) {
            const int f = i / (OY * TX), rem = i % (OY * TX);
            fo[r] = T::foff(f) + (rem / TX + N) * LXT + (rem % TX) * N;
        } else {
            const int ii = i - T::NXF;
            const int f = ii / (TY * OX), rem = ii % (TY * OX);
            fo[r] = T::foff(f) + (rem / OX) * N * LXT + rem % OX + N;
        }
    }
    auto faces = [&](int l, int buf) {
        if (!NEED_R) return;
        const double* slot = ring + (l % S) * SS;
        double* xf = XFb + buf * T::NXF;
        double* yf = YFb + buf * T::NYF;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            int i = tid + r * BLK;
            if (i < T::NXF) {
                const double* s = slot + fo[r];
                const double2 v01 = *reinterpret_cast<const double2*>(s);
                const double2 v23 = *reinterpret_cast<const double2*>(s + 2);
                double d = lt.dx[N * (N + 1) + 0] * v01.x;
                d = fma(lt.dx[N * (N + 1) + 1], v01.y, d);
                d = fma(lt.dx[N * (N + 1) + 2], v23.x, d);
                d = fma(lt.dx[N * (N + 1) + 3], v23.y, d);
                d = fma(lt.dx[N * (N + 1) + 4], s[4], d);
                xf[i] = d;
            } else if (i < T::NXF + T::NYF) {
                i -= T::NXF;
                const double* s = slot + fo[r];
                double d = lt.dy[N * (N + 1)] * s[0];
#pragma unroll
                for (int m = 1; m <= N; ++m) d = fma(lt.dy[N * (N + 1) + m], s[m * LXT], d);
                yf[i] = d;
            }
        }
    };

    double W[6][N + 1];    // the column's window: levels base .. base+N of the 6 planes
    double PLw[N + 1];     // linearised pressure G0 rho' + H0 theta' on the window
    double car[7];         // row-N partials of the layer below (bottom face)
#pragma unroll
    for (int f = 0; f < 7; ++f) car[f] = 0.0;
#pragma unroll
    for (int m = 0; m <= N; ++m) {
        PLw[m] = 0.0;
#pragma unroll
        for (int f = 0; f < 6; ++f) W[f][m] = 0.0;
    }

    mbar_wait(&mbar[0], 0);
    faces(0, 0);
    __syncthreads();

    unsigned fl = 0;   // flag bits of this thread's points (one atomic at the end)
    // one level of the sweep; KK = the level's row in the window (static: the
    // own point's values come from the window registers), N on the top level
    auto level = [&](const int l, auto kc) {
        constexpr int KK = decltype(kc)::v;
        constexpr bool top = (KK == N);
        // level parity (face-partial and staging double buffers): the layers
        // start on levels l0 = 0 mod N (N even) and the top level Z-1 = nez N
        constexpr int par = KK & 1;
        static_assert(N % 2 == 0, "static level parity");
        const long long o = colo + (long long)l * zs;
        const double* slot = ring + (l % S) * SS;
        const double* xfb = XFb + par * T::NXF;
        const double* yfb = YFb + par * T::NYF;
        double dzr[N + 1];
#pragma unroll
        for (int m = 0; m <= N; ++m) dzr[m] = lt.dzs[l][m];
        const double czf = lt.czf[l];
        const double rho0 = lt.v[C_RHO0][l];

        // the point's own state (window row KK)
        PtSt p;
        p.r = W[0][KK];
        p.u = W[1][KK];
        p.v = W[2][KK];
        p.w = W[3][KK];
        p.th = W[4][KK];
        p.rho = rho0 + p.r;
        p.rinv = NEED_R ? 1.0 / p.rho : 0.0;
        PtAcc c;
        c.R0 = c.R1 = c.R2 = c.R3 = c.R4 = c.divu = c.dwz = c.dPLz = 0.0;
#pragma unroll
        for (int f = 0; f < 6; ++f) {
            if (!NEED_R && f != 3) continue;
            double gxv = 0.0, gyv = 0.0;
            if (NEED_R) {
                const double* s = slot + T::foff(f);
                const double2 v01 = *reinterpret_cast<const double2*>(s + xo);
                const double2 v23 = *reinterpret_cast<const double2*>(s + xo + 2);
                double dx = Dxr[0] * v01.x;
                dx = fma(Dxr[1], v01.y, dx);
                dx = fma(Dxr[2], v23.x, dx);
                dx = fma(Dxr[3], v23.y, dx);
                dx = fma(Dxr[4], s[xo + 4], dx);
                gxv = fma(fxs, xfb[f * (OY * TX) + xfo], dx);
                double dy = Dyr[0] * s[yo];
#pragma unroll
                for (int m = 1; m <= N; ++m) dy = fma(Dyr[m], s[yo + m * LXT], dy);
                gyv = fma(fys, yfb[f * (TY * OX) + yfo], dy);
            }
            double dz = dzr[0] * W[f][0];
#pragma unroll
            for (int m = 1; m <= N; ++m) dz = fma(dzr[m], W[f][m], dz);
            ec_fold(f, gxv, gyv, fma(czf, car[f], dz), p, c);
        }
        if (NEED_L) {
            double dz = dzr[0] * PLw[0];
#pragma unroll
            for (int m = 1; m <= N; ++m) dz = fma(dzr[m], PLw[m], dz);
            ec_fold(6, 0.0, 0.0, fma(czf, car[6], dz), p, c);
        }
        {
            // every thread computes; only owned points store or raise flags
            if (NEED_R) fl |= own ? ec_bits(a, p, lt.v[C_TH0][l]) : 0u;
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
            ec_finish<MODE>(p, c, rho0, lt.v[C_DRHO0][l], lt.v[C_DTH0][l], lt.v[C_IRHO0][l], gr, bx, by,
                            (l == 0) || top, Rv, Lv);
            if (T::NOUT) {
                // imexcore.py:398-403, 409-411: P, Quv by plain stores, A and F staged
                const double dt = a.dt;
                const double qv[5] = {p.r, p.u, p.v, p.w, p.th};
                double* so = sOut + par * (T::NOUT * OX * OY) + tid;
                double pr[5];
#pragma unroll
                for (int f = 0; f < 5; ++f) {
                    pr[f] = qv[f] + dt * (a.a_p * (Rv[f] - Lv[f]) + a.at_p * Lv[f]);
                    so[f * OX * OY] = qv[f] + dt * (a.a_a * (Rv[f] - Lv[f]) + a.at_a * Lv[f]);
                    so[(5 + f) * OX * OY] = qv[f] + a.cb * Rv[f];
                }
                const long long fs = g.fs;
                if (own) {
                    a.P[o] = pr[0];
                    a.P[o + 3 * fs] = pr[3];
                    a.P[o + 4 * fs] = pr[4];
                    a.Quv[o + fs] = bx ? 0.0 : pr[1];
                    a.Quv[o + 2 * fs] = by ? 0.0 : pr[2];
                }
            } else {
                ec_epilogue<MODE>(a, lt, o, l, p, Rv, Lv, Ai, Fi, bx, by, own, &fl);
            }
        }
        if (l + 1 < Z) faces(l + 1, par ^ 1);
        if (T::NOUT) {
            // staged outputs visible to the async proxy; the store that read
            // the other staging buffer (level l-1) has finished reading it
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        __syncthreads();
        if (T::NOUT && tid == 0) {
            const double* so = sOut + par * (T::NOUT * OX * OY);
            tma_store_4d(&tmO0, so, ax0, ay0, l, 0);                  // A
            tma_store_4d(&tmO1, so + 5 * OX * OY, ax0, ay0, l, 0);    // F
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        // refills of the slots level l used; the issuing warp rotates so the
        // issue latency does not always fall on the same warp
        if (tid == 32 * (l % (BLK / 32)) && (l + S < Z || (T::NAF && l + T::SAF < Z))) {
            // generic-proxy reads of the slots are ordered before their async-proxy refill
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (l + S < Z) issue(l + S);
            if (T::NAF && l + T::SAF < Z) issue_af(l + T::SAF);
        }
    };
    // element layers: the window (levels l0 .. l0+N) is loaded at the layer start
    for (int l0 = 0; l0 + 1 < Z; l0 += N) {
        const int l = l0;
        if (l > 0) {
            // carries of the finished layer (row N of its element)
#pragma unroll
            for (int f = 0; f < 6; ++f) {
                double c = lt.dz[N * (N + 1)] * W[f][0];
#pragma unroll
                for (int m = 1; m <= N; ++m) c = fma(lt.dz[N * (N + 1) + m], W[f][m], c);
                car[f] = c;
            }
            if (NEED_L) {
                double c = lt.dz[N * (N + 1)] * PLw[0];
#pragma unroll
                for (int m = 1; m <= N; ++m) c = fma(lt.dz[N * (N + 1) + m], PLw[m], c);
                car[6] = c;
            }
        }
#pragma unroll
        for (int m = 1; m <= N; ++m) mbar_wait(&mbar[(l + m) % S], ((l + m) / S) & 1);
#pragma unroll
        for (int m = 0; m <= N; ++m) {
            const double* sp = ring + ((l + m) % S) * SS + po;
#pragma unroll
            for (int f = 0; f < 6; ++f) W[f][m] = sp[T::foff(f)];
            if (NEED_L) PLw[m] = lt.v[C_G0][l + m] * W[0][m] + lt.v[C_H0][l + m] * W[4][m];
        }
        level(l0, KI<0>{});
        level(l0 + 1, KI<1>{});
        level(l0 + 2, KI<2>{});
        level(l0 + 3, KI<3>{});
    }
    level(Z - 1, KI<N>{});
    if (fl) atomicOr(a.flags, fl);
    if (T::NOUT && tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#ifdef HEVI_EDGE_TIMING
    if (tid == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        atomicMax(a.dbg + 2, t);
        // the end of the tiles before the last partial wave (148 SMs; tools/tail_timing.py)
        const unsigned nb = gridDim.x * gridDim.y, b = blockIdx.x + blockIdx.y * gridDim.x;
        if (b < nb - nb % 148u) atomicMax(a.dbg + 5, t);
    }
#endif
}

// end of a domain-end kernel launched as a programmatic dependent of the
// sweep: the grid completes only after the sweep has (the stream work that
// follows reads both); a no-op for an ordinary launch
__device__ __forceinline__ void ec_edge_done() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// the domain-end planes x = X-1 / y = Y-1 inside the rank's ownership: one
// thread per point, element lines read from global memory (L2)
template <int N>
__device__ __forceinline__ double ec_gline(const double* f, long long off, long long stride,
                                           const double* Drow) {
    double d = Drow[0] * f[off];
#pragma unroll
    for (int m = 1; m <= N; ++m) d = fma(Drow[m], f[off + m * stride], d);
    return d;
}

template <int N, int MODE>
__global__ void __launch_bounds__(128) k_ecol_edge(const EArgs a, const __grid_constant__ LvlTab lt,
                                                   int nxc, int nyr, int xlo, int ylo) {
    constexpr bool NEED_L = (MODE == M_L || MODE == M_S1 || MODE == M_S2);
    constexpr bool NEED_R = (MODE != M_L);
    const Geo& G = a.g;
    // points: nxc column points (x = X-1, y = ylo ..), then nyr row points (y = Y-1, x = xlo ..), per level
    const long long per = (long long)nxc + nyr;
    const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
#ifdef HEVI_EDGE_TIMING
    if (threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        atomicMax(a.dbg + 3, ~0ull - t);
    }
#endif
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
    const long long fs = G.fs;
    const long long zs = (long long)G.lY * G.px;
    const int ix = gx - G.x0, iy = gy - G.y0;
    const long long o = (long long)gz * zs + (long long)iy * G.px + ix;
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
    double Dxr[N + 1], Dyr[N + 1], Dzr[N + 1], DxN[N + 1], DyN[N + 1], DzN[N + 1];
#pragma unroll
    for (int m = 0; m <= N; ++m) {
        Dxr[m] = lt.dx[rxw * (N + 1) + m];
        DxN[m] = lt.dx[N * (N + 1) + m];
        Dyr[m] = lt.dy[ryw * (N + 1) + m];
        DyN[m] = lt.dy[N * (N + 1) + m];
        Dzr[m] = lt.dz[rzw * (N + 1) + m];
        DzN[m] = lt.dz[N * (N + 1) + m];
    }
    const double cxv = __ldg(a.cx + gx), cyv = __ldg(a.cy + gy), czv = lt.v[C_CZ][gz];
    const long long xl = (long long)gz * zs + (long long)iy * G.px + (sx - G.x0);
    const long long xll = xl - N;
    const long long yl = (long long)gz * zs + (long long)(sy - G.y0) * G.px + ix;
    const long long yll = yl - (long long)N * G.px;
    const long long zl = (long long)sz * zs + (long long)iy * G.px + ix;
    const long long zll = zl - (long long)N * zs;
    const double* q = a.q;
    const double rho0 = lt.v[C_RHO0][gz];
    PtSt p;
    p.r = q[o];
    p.u = q[o + fs];
    p.v = q[o + 2 * fs];
    p.w = q[o + 3 * fs];
    p.th = q[o + 4 * fs];
    p.rho = rho0 + p.r;
    p.rinv = NEED_R ? 1.0 / p.rho : 0.0;
    PtAcc c;
    c.R0 = c.R1 = c.R2 = c.R3 = c.R4 = c.divu = c.dwz = c.dPLz = 0.0;
#pragma unroll
    for (int f = 0; f < 6; ++f) {
        if (!NEED_R && f != 3) continue;
        const double* F = f < 5 ? q + f * fs : a.pp_in;
        double gxv = 0.0, gyv = 0.0;
        if (NEED_R) {
            double dx = ec_gline<N>(F, xl, 1, Dxr);
            if (fx) dx += ec_gline<N>(F, xll, 1, DxN);
            gxv = cxv * dx;
            double dy = ec_gline<N>(F, yl, G.px, Dyr);
            if (fy) dy += ec_gline<N>(F, yll, G.px, DyN);
            gyv = cyv * dy;
        }
        double dz = ec_gline<N>(F, zl, zs, Dzr);
        if (fz) dz += ec_gline<N>(F, zll, zs, DzN);
        ec_fold(f, gxv, gyv, czv * dz, p, c);
    }
    if (NEED_L) {
        auto pl = [&](long long off, int lz) {
            return lt.v[C_G0][lz] * q[off] + lt.v[C_H0][lz] * q[off + 4 * fs];
        };
        double dz = Dzr[0] * pl(zl, sz);
#pragma unroll
        for (int m = 1; m <= N; ++m) dz = fma(Dzr[m], pl(zl + m * zs, sz + m), dz);
        if (fz) {
            double e = DzN[0] * pl(zll, sz - N);
#pragma unroll
            for (int m = 1; m <= N; ++m) e = fma(DzN[m], pl(zll + m * zs, sz - N + m), e);
            dz += e;
        }
        ec_fold(6, 0.0, 0.0, czv * dz, p, c);
    }
    if (NEED_R) ec_check(a, p, lt.v[C_TH0][gz]);
    const bool bx = (gx == 0) || (gx == G.X - 1);
    const bool by = (gy == 0) || (gy == G.Y - 1);
    const bool bz = (gz == 0) || (gz == G.Z - 1);
    double Rv[5], Lv[5];
    ec_finish<MODE>(p, c, rho0, lt.v[C_DRHO0][gz], lt.v[C_DTH0][gz], lt.v[C_IRHO0][gz], a.ph.g, bx, by, bz,
                    Rv, Lv);
    double Ai[5] = {0, 0, 0, 0, 0}, Fi[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int f = 0; f < 5; ++f) {
        if (MODE == M_S2) Ai[f] = a.A[o + f * fs];
        if (MODE == M_S2 || MODE == M_S3) Fi[f] = a.F[o + f * fs];
    }
    ec_epilogue<MODE>(a, lt, o, gz, p, Rv, Lv, Ai, Fi, bx, by);
#ifdef HEVI_EDGE_TIMING
    {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        atomicMax(a.dbg + 4, t);
    }
#endif
    ec_edge_done();
}
