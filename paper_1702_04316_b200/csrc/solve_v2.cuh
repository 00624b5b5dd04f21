// solve_v2.cuh -- production column kernel (included by hevi.cu inside its
// anonymous namespace).
//
// One thread per vertical column, fused:
//   forward  (bottom -> top, one element of N levels per iteration):
//     Schur RHS  Pe - lam (F0 ua + rho0 G0 d/dz ua)   (imexcore.py:229-243)
//     and forward substitution with L                 (columnsolve.py:172-174)
//   backward (top -> bottom):
//     back substitution with U                        (columnsolve.py:176-180)
//     and, one element behind, the extraction of w, theta', rho'
//                                                     (imexcore.py:273-287)
// The element's ua / y / x values live in register windows (static indices
// after unrolling), the forward results y in shared memory; the band LU
// (shared by all columns on box meshes) is read from shared memory with a
// fixed width of 2N sub/super-diagonals (the Schur column bandwidth is 2N+1).
#pragma once

struct S2Args {
    Geo g;
    Phys ph;
    const double* tab;   // 12 x M level tables (see k_lu_dense2 / plan)
    const double* LU2;   // M x (4N+1), d = j - k + 2N
    const double* rU;    // 1/U_kk
    const double* Dz;
    int ainv_identity;
    double lam;
    const double* P;       // predictor fields 0,3,4
    double* out;           // writes fields 0,3,4
    const double* src_uv;  // optional: copy u,v (with no-flux zeroing)
    double* pp_out;        // optional (set2nc): P' of the solved state (next explicit stage reads it)
    const double* rec;     // k_solve2's per-level records (k_s2rec)
    Lev lv;
    double bc[16];
    double Dzc[81];        // the D matrix in the parameter bank (k_solve2: static indices)
};

// P' of a solved point: the explicit kernel's pprime (explicit_v2.cuh) on the
// same inputs, written once here instead of per staged point downstream
// PT: the level's [rho0 | theta0 | 1/(rho0 theta0) | Pb | Pb - P0f | P0f]
__device__ __forceinline__ double solved_pprime(const S2Args& a, const double* PT, double r, double th) {
    const double rho0 = PT[0], th0 = PT[1];
    const double delta = (r * th0 + th * (rho0 + r)) * PT[2];
    if (HEVI_PP_SHORT && fabs(delta) <= 0x1p-10) {
        // |delta| <= 2^-10: the terms beyond delta^6 are below 1e-20 relative
        double s = a.bc[5];
#pragma unroll
        for (int j = 4; j >= 0; --j) s = fma(s, delta, a.bc[j]);
        return fma(PT[3], s * delta, PT[4]);
    }
    if (fabs(delta) <= 0.125) {
        double s = a.bc[14];
#pragma unroll
        for (int j = 13; j >= 0; --j) s = fma(s, delta, a.bc[j]);
        return fma(PT[3], s * delta, PT[4]);
    }
    return pprime_pow(rho0 + r, th0 + th, PT[5], a.ph.P0, a.ph.R, a.ph.gamma);
}

enum { V_G0 = 0, V_H0, V_F0Z, V_RG, V_CZ, V_COEF, V_UA, V_DEN, V_DTH0, V_IRHO0, V_IG0R, V_IG0,
       V_F0C, V_TH0, V_IFT, V_ITH0, V_NT };

// P' level tables of the pivoted kernel: [6][M]
__device__ __forceinline__ void load_pp_tables(const S2Args& a, double* PT, int M, int tid, int T) {
    const Lev& lv = a.lv;
    for (int i = tid; i < M; i += T) {
        PT[i] = lv.rho0[i];
        PT[M + i] = lv.theta0[i];
        PT[2 * M + i] = lv.irt0[i];
        PT[3 * M + i] = lv.E0[i];
        PT[4 * M + i] = lv.c0[i];
        PT[5 * M + i] = lv.P0f[i];
    }
}

// k_solve2's per-level record in shared memory: everything a level of the
// sweeps reads, at immediate offsets from one base register per element
//   [0, 2N)        L row (sub-diagonals, d = 2N - j for j = 1 .. 2N)
//   2N             1 / U_kk
//   [2N+2, 4N+2)   U row (super-diagonals j = 1 .. 2N)
//   [4N+2, +V_NT)  the Schur / extraction level tables (V_*)
//   then 6         P' tables (solved_pprime)
template <int N>
struct S2Rec {
    static constexpr int L = 0, RU = 2 * N, U = 2 * N + 2, TB = 4 * N + 2, PT = TB + (V_NT + 1) / 2 * 2;
    static constexpr int RS = PT + 6;   // even: every record 16-byte aligned
    static_assert(RS % 2 == 0, "record stride");
};

// the records of a factor, built once per lam (runtime N; layout as S2Rec<N>)
__global__ void k_s2rec(const double* __restrict__ LU2, const double* __restrict__ rU,
                        const double* __restrict__ tab, const Lev lv, int M, int N, double* rec) {
    const int W = 4 * N + 1, RU = 2 * N, U = 2 * N + 2, TB = 4 * N + 2, PT = TB + (V_NT + 1) / 2 * 2;
    const int RS = PT + 6;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < M * RS; i += gridDim.x * blockDim.x) {
        const int k = i / RS, j = i - k * RS;
        double v = 0.0;
        if (j < 2 * N) v = LU2[k * W + j];                                // L: d = j
        else if (j == RU) v = rU[k];
        else if (j >= U && j < U + 2 * N) v = LU2[k * W + 2 * N + 1 + (j - U)];
        else if (j >= TB && j < TB + V_NT) v = tab[(j - TB) * M + k];
        else if (j >= PT) {
            const int t = j - PT;
            v = t == 0 ? lv.rho0[k] : t == 1 ? lv.theta0[k] : t == 2 ? lv.irt0[k]
              : t == 3 ? lv.E0[k] : t == 4 ? lv.c0[k] : lv.P0f[k];
        }
        rec[i] = v;
    }
}

template <int N>
__host__ __device__ constexpr size_t s2_smem_bytes(int M, int T) {
    return sizeof(double) * ((size_t)M * S2Rec<N>::RS + (size_t)(N + 1) * (N + 1) + (size_t)M * T);
}

// L2 prefetch distance (elements) of the column sweeps: the next element's
// lines are requested while this element is substituted (0.294 -> 0.257 ms
// per solve at config 5; distance 2 measured slower)
#ifndef HEVI_S2_PF
#define HEVI_S2_PF 2
#endif

template <int N, bool SC>   // SC: conservative set set2c
// (128, 3): at most 168 registers, 12 warps per SM (3 per scheduler: the
// register file is split 16 K per sub-partition) -- faster than the
// 128-register, 16-warp schedule of __launch_bounds__(128) (0.2975 -> 0.288
// ms per solve) and, with the backward lines loaded one element ahead, than
// the 184-register, 8-warp schedule that look-ahead takes unbounded (0.274
// vs 0.325 ms)
__global__ void __launch_bounds__(128, 3) k_solve2(const S2Args a) {
    using R = S2Rec<N>;
    constexpr int RS = R::RS;
    extern __shared__ __align__(16) double sm2[];
    const Geo& g = a.g;
    const int M = g.Z;
    const int T = blockDim.x;
    const int tid = threadIdx.x;
    double* rec = sm2;                        // M * RS
    double* sD = rec + (size_t)M * RS;        // (N+1)^2 (set2c)
    double* Y = sD + (N + 1) * (N + 1);       // M * T
    // the vertical D matrix: set2nc reads the parameter bank (static indices,
    // no shared loads: -1.4 % per solve); set2c keeps shared memory (the
    // parameter-bank form measured 8 % slower there)
#define DZC(i) (SC ? sD[i] : a.Dzc[i])
    {
        const double2* src = reinterpret_cast<const double2*>(a.rec);
        double2* dst = reinterpret_cast<double2*>(rec);
        for (int i = tid; i < M * RS / 2; i += T) dst[i] = src[i];
    }
    if (SC)
        for (int i = tid; i < (N + 1) * (N + 1); i += T) sD[i] = a.Dz[i];
    __syncthreads();

    const int NYo = g.slab ? 1 : N;
    const int xlo = g.ex_b * N;
    const int cntx = (g.ex_e - g.ex_b) * N + (g.ex_e == g.nex ? 1 : 0);
    const int ylo = g.ey_b * NYo;
    const int cnty = (g.ey_e - g.ey_b) * NYo + (g.ey_e == g.ney ? 1 : 0);
    const int ncol = cntx * cnty;
    // persistent CTAs: the record prologue once per CTA, column blocks strided
    for (int cb = blockIdx.x * T; cb < ncol; cb += gridDim.x * T) {
    const int c = cb + tid;
    if (c >= ncol) break;
    const int gx = xlo + c % cntx;
    const int gy = ylo + c / cntx;
    const int gys = g.slab ? 0 : gy;
    const long long fs = g.fs;
    const double lam = a.lam, gr = a.ph.g;
    const bool ident = a.ainv_identity != 0;
    const int nez = g.nez;
    // per-field column bases; level k of a field at base[k * ls] (32-bit offsets)
    const double* Ps = a.P + loff(g, gx, gys, 0);   // source column (slab: y = 0)
    const double* Ps3 = Ps + 3 * fs;
    const double* Ps4 = Ps + 4 * fs;
    const double* Po = a.P + loff(g, gx, gy, 0);    // own column
    const double* Po3 = Po + 3 * fs;
    const double* Po4 = Po + 4 * fs;
    double* Oo = a.out + loff(g, gx, gy, 0);
    double* Oo3 = Oo + 3 * fs;
    double* Oo4 = Oo + 4 * fs;
    double* PPo = a.pp_out ? a.pp_out + loff(g, gx, gy, 0) : nullptr;
    const int ls = g.lY * g.px;                     // level stride
    double* Yt = Y + tid;
#define TBk(rk, t) (rk)[R::TB + (t)]

    // ua_z of the Schur RHS (imexcore.py:236-240); `re` only enters set2c
    auto ua_of2 = [&](const double* rk, double re, double we, double te, int k) -> double {
        double v = SC ? we - (lam * (re - te * TBk(rk, V_ITH0))) * gr : we + (TBk(rk, V_COEF) * te) * gr;
        if (!ident) v = v - TBk(rk, V_UA) * ((TBk(rk, V_DTH0) * v) / TBk(rk, V_DEN));
        return (k == 0 || k == M - 1) ? 0.0 : v;
    };

    // ---------------- forward: RHS + L substitution --------------------------
    double uaw[N + 1], Pew[N + 1], yw[3 * N];
#pragma unroll
    for (int i = 0; i < 3 * N; ++i) yw[i] = 0.0;
    {
        const double re = Ps[0], we = Ps3[0], te = Ps4[0];
        uaw[0] = ua_of2(rec, re, we, te, 0);
        Pew[0] = SC ? TBk(rec, V_F0C) * te : TBk(rec, V_G0) * re + TBk(rec, V_H0) * te;
    }
    double carry = 0.0;
    double re[N], we[N], te[N];   // predictor lines of the current element (levels k0+1 .. k0+N)
    {
        int o = ls;
#pragma unroll
        for (int l = 1; l <= N; ++l, o += ls) {
            re[l - 1] = Ps[o];
            we[l - 1] = Ps3[o];
            te[l - 1] = Ps4[o];
        }
    }
    for (int e = 0; e < nez; ++e) {
        const int k0 = e * N;
        const double* r0 = rec + k0 * RS;      // level k0 + l at r0 + l * RS
        double* Yk = Yt + k0 * T;              // level k0 + l at Yk[l * T]
        const int o1 = (k0 + 1) * ls;
        if (HEVI_S2_PF && e + HEVI_S2_PF < nez) {   // a later element's lines into L2
            int o = o1 + HEVI_S2_PF * N * ls;
#pragma unroll
            for (int l = 1; l <= N; ++l, o += ls) {
                pf_l2(Ps + o);
                pf_l2(Ps3 + o);
                pf_l2(Ps4 + o);
            }
        }
#pragma unroll
        for (int l = 1; l <= N; ++l) {
            const double* rk = r0 + l * RS;
            uaw[l] = ua_of2(rk, re[l - 1], we[l - 1], te[l - 1], k0 + l);
            Pew[l] = SC ? TBk(rk, V_F0C) * te[l - 1] : TBk(rk, V_G0) * re[l - 1] + TBk(rk, V_H0) * te[l - 1];
        }
        // the next element's predictor lines, in flight during this element's substitution
        if (e + 1 < nez) {
            int o = o1 + N * ls;
#pragma unroll
            for (int l = 1; l <= N; ++l, o += ls) {
                re[l - 1] = Ps[o];
                we[l - 1] = Ps3[o];
                te[l - 1] = Ps4[o];
            }
        }
#pragma unroll
        for (int l = 0; l < N; ++l) {
            const double* rk = r0 + l * RS;
            double d = 0.0;
#pragma unroll
            for (int m = 0; m <= N; ++m) d = fma(DZC(l * (N + 1) + m), uaw[m], d);
            if (l == 0 && e > 0) d += carry;
            const double dua = TBk(rk, V_CZ) * d;
            // imexcore._helmholtz_flux (imexcore.py:263-268)
            const double rhs = SC ? Pew[l] - TBk(rk, V_F0C) * lam * (TBk(rk, V_TH0) * dua + TBk(rk, V_DTH0) * uaw[l])
                                  : Pew[l] - lam * (TBk(rk, V_F0Z) * uaw[l] + TBk(rk, V_RG) * dua);
            double s = 0.0;
#pragma unroll
            for (int j = 1; j <= 2 * N; ++j) s = fma(rk[R::L + 2 * N - j], yw[2 * N + l - j], s);
            const double y = rhs - s;
            yw[2 * N + l] = y;
            Yk[l * T] = y;
        }
        // row N of this element: the lower half of the next face derivative
        double cr = 0.0;
#pragma unroll
        for (int m = 0; m <= N; ++m) cr = fma(DZC(N * (N + 1) + m), uaw[m], cr);
        carry = cr;
        if (e + 1 < nez) {
#pragma unroll
            for (int i = 0; i < 2 * N; ++i) yw[i] = yw[i + N];
            uaw[0] = uaw[N];
            Pew[0] = Pew[N];
        }
    }
    {   // top level: row N of the last element, boundary
        const int k = M - 1;
        const double* rk = rec + k * RS;
        const double dua = TBk(rk, V_CZ) * carry;
        const double rhs = SC ? Pew[N] - TBk(rk, V_F0C) * lam * (TBk(rk, V_TH0) * dua + TBk(rk, V_DTH0) * uaw[N])
                              : Pew[N] - lam * (TBk(rk, V_F0Z) * uaw[N] + TBk(rk, V_RG) * dua);
        double s = 0.0;
#pragma unroll
        for (int j = 1; j <= 2 * N; ++j) s = fma(rk[R::L + 2 * N - j], yw[3 * N - j], s);
        Yt[k * T] = rhs - s;
    }

    // ---------------- backward: U substitution + extraction -------------------
    // xw[l] = x_{k0 + l}, l = 0 .. 3N (current element and 2N levels above)
    double xw[3 * N + 1];
#pragma unroll
    for (int i = 0; i <= 3 * N; ++i) xw[i] = 0.0;
    xw[N] = Yt[(M - 1) * T] * rec[(M - 1) * RS + R::RU];

    auto extract = [&](const double* rk, int k, int o, double Pk, double dsum, double re, double we,
                       double te) {
        const bool bz = (k == 0) || (k == M - 1);
        const double dP = TBk(rk, V_CZ) * dsum;
        // imexcore._up (imexcore.py:245-257)
        double up = SC ? lam * (dP + (Pk * TBk(rk, V_IFT)) * gr)
                       : lam * (dP * TBk(rk, V_IRHO0) + (Pk * TBk(rk, V_IG0R)) * gr);
        double ua = SC ? we - (lam * (re - te * TBk(rk, V_ITH0))) * gr : we + (TBk(rk, V_COEF) * te) * gr;
        if (!ident) {
            ua = ua - TBk(rk, V_UA) * ((TBk(rk, V_DTH0) * ua) / TBk(rk, V_DEN));
            up = up - TBk(rk, V_UA) * ((TBk(rk, V_DTH0) * up) / TBk(rk, V_DEN));
        }
        if (bz) {
            ua = 0.0;
            up = 0.0;
        }
        const double w = ua - up;
        double th, rho;
        if (SC) {   // imexcore.py:288-297
            th = Pk / TBk(rk, V_F0C);
            rho = ((Pk * TBk(rk, V_IFT) + (lam * TBk(rk, V_ITH0)) * (w * TBk(rk, V_DTH0))) - te * TBk(rk, V_ITH0)) + re;
        } else {    // imexcore.py:280-287
            th = te - lam * (w * TBk(rk, V_DTH0));
            rho = (Pk - TBk(rk, V_H0) * th) * TBk(rk, V_IG0);
        }
        Oo[o] = rho;
        Oo3[o] = w;
        Oo4[o] = th;
        if (!SC && PPo) PPo[o] = solved_pprime(a, rk + R::PT, rho, th);
        if (a.src_uv) {
            const bool bx = (gx == 0) || (gx == g.X - 1);
            const bool by = g.slab || (gy == 0) || (gy == g.Y - 1);
            const double* su = a.src_uv + loff(g, gx, gy, k);
            Oo[o + fs] = bx ? 0.0 : su[fs];
            Oo[o + 2 * fs] = by ? 0.0 : su[2 * fs];
        }
    };

    // the extraction's predictor lines of an element, loaded one element
    // ahead (in flight during the element above's substitution)
    double wn[N], tn[N], rn[N];
    auto load_bwd = [&](int e) {
        int o = (e * N + 1) * ls;
#pragma unroll
        for (int l = 1; l <= N; ++l, o += ls) {
            wn[l - 1] = Po3[o];
            tn[l - 1] = Po4[o];
            rn[l - 1] = SC ? Po[o] : 0.0;
        }
    };
    load_bwd(nez - 1);
    for (int e = nez - 1; e >= 0; --e) {
        const int k0 = e * N;
        const double* r0 = rec + k0 * RS;
        const double* Yk = Yt + k0 * T;
        const int o1 = (k0 + 1) * ls;
        if (HEVI_S2_PF && e >= HEVI_S2_PF) {   // an element below, into L2
            int o = o1 - HEVI_S2_PF * N * ls;
#pragma unroll
            for (int l = 1; l <= N; ++l, o += ls) {
                pf_l2(Po3 + o);
                pf_l2(Po4 + o);
                if (SC) pf_l2(Po + o);
            }
        }
        double we[N], te[N], ro[N];
#pragma unroll
        for (int l = 0; l < N; ++l) {
            we[l] = wn[l];
            te[l] = tn[l];
            ro[l] = rn[l];
        }
        if (e > 0) load_bwd(e - 1);
#pragma unroll
        for (int l = N - 1; l >= 0; --l) {
            const double* rk = r0 + l * RS;
            double s = 0.0;
#pragma unroll
            for (int j = 1; j <= 2 * N; ++j) s = fma(rk[R::U + j - 1], xw[l + j], s);
            xw[l] = (Yk[l * T] - s) * rk[R::RU];
        }
        // extraction of levels k0+1 .. k0+N (element e now complete)
        {
            int o = o1;
#pragma unroll
            for (int l = 1; l <= N; ++l, o += ls) {
                double d = 0.0;
#pragma unroll
                for (int m = 0; m <= N; ++m) d = fma(DZC(l * (N + 1) + m), xw[m], d);
                if (l == N && e + 1 < nez) {
                    double d2 = 0.0;
#pragma unroll
                    for (int m = 0; m <= N; ++m) d2 = fma(DZC(m), xw[N + m], d2);
                    d += d2;
                }
                extract(r0 + l * RS, k0 + l, o, xw[l], d, ro[l - 1], we[l - 1], te[l - 1]);
            }
        }
        if (e > 0) {
#pragma unroll
            for (int i = 2 * N; i >= 0; --i) xw[N + i] = xw[i];
        }
    }
    {   // bottom level: row 0 of element 0, boundary
        double d = 0.0;
#pragma unroll
        for (int m = 0; m <= N; ++m) d = fma(DZC(m), xw[m], d);
        extract(rec, 0, 0, xw[0], d, SC ? Po[0] : 0.0, Po3[0], Po4[0]);
    }
    }   // column blocks
#undef TBk
#undef DZC
}

// ---------------------------------------------------------------------------
// Pivoted fallback of the fused column solve (columnsolve.py:141-167): the
// shared column matrix carries a partial-pivoting dense LU (k_lu_pivot) when
// the no-pivot banded LU hits a degenerate diagonal.  One thread per column:
// Schur RHS of every level into shared memory, row interchanges, dense L and
// U substitution (scipy.linalg.lu_solve), then the same extraction as
// k_solve2.  Arguments as S2Args with LU2 = the M x M pivoted factor and
// piv its interchanges.
// ---------------------------------------------------------------------------
template <int N, bool SC>
__global__ void __launch_bounds__(128) k_solve_piv(const S2Args a, const int* __restrict__ piv) {
    extern __shared__ __align__(16) double smp[];
    const Geo& g = a.g;
    const int M = g.Z;
    const int T = blockDim.x;
    const int tid = threadIdx.x;
    double* tb = smp;                   // V_NT * M
    double* LU = tb + V_NT * M;         // M * M
    double* sD = LU + M * M;            // (N+1)^2
    double* PT = sD + (N + 1) * (N + 1); // 6 * M
    double* Y = PT + 6 * M;             // M * T
    int* sp = reinterpret_cast<int*>(Y + (size_t)M * T);   // M
    for (int i = tid; i < V_NT * M; i += T) tb[i] = a.tab[i];
    for (int i = tid; i < M * M; i += T) LU[i] = a.LU2[i];
    for (int i = tid; i < (N + 1) * (N + 1); i += T) sD[i] = a.Dz[i];
    for (int i = tid; i < M; i += T) sp[i] = piv[i];
    load_pp_tables(a, PT, M, tid, T);
    __syncthreads();

    const int NYo = g.slab ? 1 : N;
    const int xlo = g.ex_b * N;
    const int cntx = (g.ex_e - g.ex_b) * N + (g.ex_e == g.nex ? 1 : 0);
    const int ylo = g.ey_b * NYo;
    const int cnty = (g.ey_e - g.ey_b) * NYo + (g.ey_e == g.ney ? 1 : 0);
    const int c = blockIdx.x * T + tid;
    if (c >= cntx * cnty) return;
    const int gx = xlo + c % cntx;
    const int gy = ylo + c / cntx;
    const int gys = g.slab ? 0 : gy;
    const long long fs = g.fs;
    const double lam = a.lam, gr = a.ph.g;
    const bool ident = a.ainv_identity != 0;
    const int nez = g.nez;
    const double* Ps = a.P + loff(g, gx, gys, 0);
    const double* Po = a.P + loff(g, gx, gy, 0);
    double* Oo = a.out + loff(g, gx, gy, 0);
    const long long ls = (long long)g.lY * g.px;
#define TB(t, k) tb[(t) * M + (k)]
#define YY(k) Y[(size_t)(k) * T + tid]
    auto ua_at = [&](int k, const double* src) -> double {
        const long long o = (long long)k * ls;
        const double re = src[o], we = src[o + 3 * fs], te = src[o + 4 * fs];
        double v = SC ? we - (lam * (re - te * TB(V_ITH0, k))) * gr : we + (TB(V_COEF, k) * te) * gr;
        if (!ident) v = v - TB(V_UA, k) * ((TB(V_DTH0, k) * v) / TB(V_DEN, k));
        return (k == 0 || k == M - 1) ? 0.0 : v;
    };
    // folded z-derivative at level k of a per-level quantity f(k') (DSS across element faces)
    auto dz_at = [&](int k, auto&& f) -> double {
        const int e = (k == M - 1) ? nez - 1 : k / N;
        const int l = k - e * N;
        double d = 0.0;
        for (int m = 0; m <= N; ++m) d = fma(sD[l * (N + 1) + m], f(e * N + m), d);
        if (l == 0 && e > 0) {
            double d2 = 0.0;
            for (int m = 0; m <= N; ++m) d2 = fma(sD[N * (N + 1) + m], f((e - 1) * N + m), d2);
            d += d2;
        }
        return d;
    };
    // 1. Schur RHS (imexcore.py:229-243, _helmholtz_flux :259-268) of every level
    for (int k = 0; k < M; ++k) {
        const long long o = (long long)k * ls;
        const double re = Ps[o], te = Ps[o + 4 * fs];
        const double ua = ua_at(k, Ps);
        const double dua = TB(V_CZ, k) * dz_at(k, [&](int kk) { return ua_at(kk, Ps); });
        const double Pe = SC ? TB(V_F0C, k) * te : TB(V_G0, k) * re + TB(V_H0, k) * te;
        YY(k) = SC ? Pe - TB(V_F0C, k) * lam * (TB(V_TH0, k) * dua + TB(V_DTH0, k) * ua)
                   : Pe - lam * (TB(V_F0Z, k) * ua + TB(V_RG, k) * dua);
    }
    // 2. interchanges, unit-lower and upper substitution
    for (int i = 0; i < M; ++i) {
        const int p = sp[i];
        if (p != i) {
            const double t = YY(i);
            YY(i) = YY(p);
            YY(p) = t;
        }
    }
    for (int i = 1; i < M; ++i) {
        double s = 0.0;
        for (int j = 0; j < i; ++j) s = fma(LU[i * M + j], YY(j), s);
        YY(i) = YY(i) - s;
    }
    for (int i = M - 1; i >= 0; --i) {
        double s = 0.0;
        for (int j = i + 1; j < M; ++j) s = fma(LU[i * M + j], YY(j), s);
        YY(i) = (YY(i) - s) / LU[i * M + i];
    }
    // 3. extraction of w, theta', rho' (imexcore.py:245-298), as k_solve2
    for (int k = 0; k < M; ++k) {
        const long long o = (long long)k * ls;
        const double re = Po[o], we = Po[o + 3 * fs], te = Po[o + 4 * fs];
        const double Pk = YY(k);
        const bool bz = (k == 0) || (k == M - 1);
        const double dP = TB(V_CZ, k) * dz_at(k, [&](int kk) { return YY(kk); });
        double up = SC ? lam * (dP + (Pk * TB(V_IFT, k)) * gr)
                       : lam * (dP * TB(V_IRHO0, k) + (Pk * TB(V_IG0R, k)) * gr);
        double ua = SC ? we - (lam * (re - te * TB(V_ITH0, k))) * gr : we + (TB(V_COEF, k) * te) * gr;
        if (!ident) {
            ua = ua - TB(V_UA, k) * ((TB(V_DTH0, k) * ua) / TB(V_DEN, k));
            up = up - TB(V_UA, k) * ((TB(V_DTH0, k) * up) / TB(V_DEN, k));
        }
        if (bz) {
            ua = 0.0;
            up = 0.0;
        }
        const double w = ua - up;
        double th, rho;
        if (SC) {
            th = Pk / TB(V_F0C, k);
            rho = ((Pk * TB(V_IFT, k) + (lam * TB(V_ITH0, k)) * (w * TB(V_DTH0, k))) - te * TB(V_ITH0, k)) + re;
        } else {
            th = te - lam * (w * TB(V_DTH0, k));
            rho = (Pk - TB(V_H0, k) * th) * TB(V_IG0, k);
        }
        Oo[o] = rho;
        Oo[o + 3 * fs] = w;
        Oo[o + 4 * fs] = th;
        if (!SC && a.pp_out) {
            const double pt[6] = {PT[k], PT[M + k], PT[2 * M + k], PT[3 * M + k], PT[4 * M + k], PT[5 * M + k]};
            a.pp_out[loff(g, gx, gy, 0) + o] = solved_pprime(a, pt, rho, th);
        }
        if (a.src_uv) {
            const bool bx = (gx == 0) || (gx == g.X - 1);
            const bool by = g.slab || (gy == 0) || (gy == g.Y - 1);
            const double* su = a.src_uv + loff(g, gx, gy, k);
            Oo[o + fs] = bx ? 0.0 : su[fs];
            Oo[o + 2 * fs] = by ? 0.0 : su[2 * fs];
        }
    }
#undef YY
#undef TB
}
