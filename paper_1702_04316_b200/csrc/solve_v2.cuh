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
    Lev lv;
    double bc[16];
};

// the rare |delta| > 1/8 branch of pprime, out of line (keeps the column
// kernel's register budget)
__device__ __noinline__ double pprime_pow(double rho, double theta, double P0f, double P0, double R,
                                          double gamma) {
    return P0 * pow(rho * R * theta / P0, gamma) - P0f;
}

// P' of a solved point: the explicit kernel's pprime (explicit_v2.cuh) on the
// same inputs, written once here instead of per staged point downstream
// PT: per-level [rho0 | theta0 | 1/(rho0 theta0) | Pb | Pb - P0f | P0f] in shared memory
__device__ __forceinline__ double solved_pprime(const S2Args& a, const double* PT, int M, int k,
                                                double r, double th) {
    const double rho0 = PT[k], th0 = PT[M + k];
    const double delta = (r * th0 + th * (rho0 + r)) * PT[2 * M + k];
    if (HEVI_PP_SHORT && fabs(delta) <= 0x1p-10) {
        // |delta| <= 2^-10: the terms beyond delta^6 are below 1e-20 relative
        double s = a.bc[5];
#pragma unroll
        for (int j = 4; j >= 0; --j) s = fma(s, delta, a.bc[j]);
        return fma(PT[3 * M + k], s * delta, PT[4 * M + k]);
    }
    if (fabs(delta) <= 0.125) {
        double s = a.bc[14];
#pragma unroll
        for (int j = 13; j >= 0; --j) s = fma(s, delta, a.bc[j]);
        return fma(PT[3 * M + k], s * delta, PT[4 * M + k]);
    }
    return pprime_pow(rho0 + r, th0 + th, PT[5 * M + k], a.ph.P0, a.ph.R, a.ph.gamma);
}

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

enum { V_G0 = 0, V_H0, V_F0Z, V_RG, V_CZ, V_COEF, V_UA, V_DEN, V_DTH0, V_IRHO0, V_IG0R, V_IG0,
       V_F0C, V_TH0, V_IFT, V_ITH0, V_NT };

// L2 prefetch distance (elements) of the column sweeps: the next element's
// lines are requested while this element is substituted (0.294 -> 0.257 ms
// per solve at config 5; distance 2 measured slower)
#ifndef HEVI_S2_PF
#define HEVI_S2_PF 1
#endif

template <int N, bool SC>   // SC: conservative set set2c
__global__ void __launch_bounds__(128) k_solve2(const S2Args a) {
    constexpr int W = 4 * N + 1;
    extern __shared__ __align__(16) double sm2[];
    const Geo& g = a.g;
    const int M = g.Z;
    const int T = blockDim.x;
    const int tid = threadIdx.x;
    double* tb = sm2;                  // V_NT * M
    double* LU = tb + V_NT * M;        // M * W
    double* rU = LU + M * W;           // M
    double* sD = rU + M;               // (N+1)^2
    double* PT = sD + (N + 1) * (N + 1);  // 6 * M: P' level tables
    double* Y = PT + 6 * M;            // M * T
    for (int i = tid; i < V_NT * M; i += T) tb[i] = a.tab[i];
    for (int i = tid; i < M * W; i += T) LU[i] = a.LU2[i];
    for (int i = tid; i < M; i += T) rU[i] = a.rU[i];
    for (int i = tid; i < (N + 1) * (N + 1); i += T) sD[i] = a.Dz[i];
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
    const double* Ps = a.P + loff(g, gx, gys, 0);   // source column (slab: y = 0)
    const double* Po = a.P + loff(g, gx, gy, 0);    // own column
    double* Oo = a.out + loff(g, gx, gy, 0);
    const long long ls = (long long)g.lY * g.px;    // level stride
#define TB(t, k) tb[(t) * M + (k)]

    // ua_z of the Schur RHS (imexcore.py:236-240); `re` only enters set2c
    auto ua_of2 = [&](double re, double we, double te, int k) -> double {
        double v = SC ? we - (lam * (re - te * TB(V_ITH0, k))) * gr : we + (TB(V_COEF, k) * te) * gr;
        if (!ident) v = v - TB(V_UA, k) * ((TB(V_DTH0, k) * v) / TB(V_DEN, k));
        return (k == 0 || k == M - 1) ? 0.0 : v;
    };

    // ---------------- forward: RHS + L substitution --------------------------
    double uaw[N + 1], Pew[N + 1], yw[3 * N];
#pragma unroll
    for (int i = 0; i < 3 * N; ++i) yw[i] = 0.0;
    {
        const double re = Ps[0], we = Ps[3 * fs], te = Ps[4 * fs];
        uaw[0] = ua_of2(re, we, te, 0);
        Pew[0] = SC ? TB(V_F0C, 0) * te : TB(V_G0, 0) * re + TB(V_H0, 0) * te;
    }
    double carry = 0.0;
    for (int e = 0; e < nez; ++e) {
        const int k0 = e * N;
        if (HEVI_S2_PF && e + HEVI_S2_PF < nez) {   // a later element's lines into L2
#pragma unroll
            for (int l = 1; l <= N; ++l) {
                const long long o = (long long)(k0 + HEVI_S2_PF * N + l) * ls;
                pf_l2(Ps + o);
                pf_l2(Ps + o + 3 * fs);
                pf_l2(Ps + o + 4 * fs);
            }
        }
        double re[N], we[N], te[N];
#pragma unroll
        for (int l = 1; l <= N; ++l) {
            const long long o = (long long)(k0 + l) * ls;
            re[l - 1] = Ps[o];
            we[l - 1] = Ps[o + 3 * fs];
            te[l - 1] = Ps[o + 4 * fs];
        }
#pragma unroll
        for (int l = 1; l <= N; ++l) {
            const int k = k0 + l;
            uaw[l] = ua_of2(re[l - 1], we[l - 1], te[l - 1], k);
            Pew[l] = SC ? TB(V_F0C, k) * te[l - 1] : TB(V_G0, k) * re[l - 1] + TB(V_H0, k) * te[l - 1];
        }
#pragma unroll
        for (int l = 0; l < N; ++l) {
            const int k = k0 + l;
            double d = 0.0;
#pragma unroll
            for (int m = 0; m <= N; ++m) d = fma(sD[l * (N + 1) + m], uaw[m], d);
            if (l == 0 && e > 0) d += carry;
            const double dua = TB(V_CZ, k) * d;
            // imexcore._helmholtz_flux (imexcore.py:263-268)
            const double rhs = SC ? Pew[l] - TB(V_F0C, k) * lam * (TB(V_TH0, k) * dua + TB(V_DTH0, k) * uaw[l])
                                  : Pew[l] - lam * (TB(V_F0Z, k) * uaw[l] + TB(V_RG, k) * dua);
            double s = 0.0;
            const double* Lr = LU + k * W;
#pragma unroll
            for (int j = 1; j <= 2 * N; ++j) s = fma(Lr[2 * N - j], yw[2 * N + l - j], s);
            const double y = rhs - s;
            yw[2 * N + l] = y;
            Y[k * T + tid] = y;
        }
        // row N of this element: the lower half of the next face derivative
        double cr = 0.0;
#pragma unroll
        for (int m = 0; m <= N; ++m) cr = fma(sD[N * (N + 1) + m], uaw[m], cr);
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
        const double dua = TB(V_CZ, k) * carry;
        const double rhs = SC ? Pew[N] - TB(V_F0C, k) * lam * (TB(V_TH0, k) * dua + TB(V_DTH0, k) * uaw[N])
                              : Pew[N] - lam * (TB(V_F0Z, k) * uaw[N] + TB(V_RG, k) * dua);
        double s = 0.0;
        const double* Lr = LU + k * W;
#pragma unroll
        for (int j = 1; j <= 2 * N; ++j) s = fma(Lr[2 * N - j], yw[3 * N - j], s);
        Y[k * T + tid] = rhs - s;
    }

    // ---------------- backward: U substitution + extraction -------------------
    // xw[l] = x_{k0 + l}, l = 0 .. 3N (current element and 2N levels above)
    double xw[3 * N + 1];
#pragma unroll
    for (int i = 0; i <= 3 * N; ++i) xw[i] = 0.0;
    xw[N] = Y[(M - 1) * T + tid] * rU[M - 1];

    auto extract = [&](int k, double Pk, double dsum, double re, double we, double te) {
        const bool bz = (k == 0) || (k == M - 1);
        const double dP = TB(V_CZ, k) * dsum;
        // imexcore._up (imexcore.py:245-257)
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
        if (SC) {   // imexcore.py:288-297
            th = Pk / TB(V_F0C, k);
            rho = ((Pk * TB(V_IFT, k) + (lam * TB(V_ITH0, k)) * (w * TB(V_DTH0, k))) - te * TB(V_ITH0, k)) + re;
        } else {    // imexcore.py:280-287
            th = te - lam * (w * TB(V_DTH0, k));
            rho = (Pk - TB(V_H0, k) * th) * TB(V_IG0, k);
        }
        const long long o = (long long)k * ls;
        Oo[o] = rho;
        Oo[o + 3 * fs] = w;
        Oo[o + 4 * fs] = th;
        if (!SC && a.pp_out) a.pp_out[loff(g, gx, gy, 0) + o] = solved_pprime(a, PT, M, k, rho, th);
        if (a.src_uv) {
            const bool bx = (gx == 0) || (gx == g.X - 1);
            const bool by = g.slab || (gy == 0) || (gy == g.Y - 1);
            const double* su = a.src_uv + loff(g, gx, gy, k);
            Oo[o + fs] = bx ? 0.0 : su[fs];
            Oo[o + 2 * fs] = by ? 0.0 : su[2 * fs];
        }
    };

    for (int e = nez - 1; e >= 0; --e) {
        const int k0 = e * N;
        if (HEVI_S2_PF && e >= HEVI_S2_PF) {   // an element below, into L2
#pragma unroll
            for (int l = 1; l <= N; ++l) {
                const long long o = (long long)(k0 - HEVI_S2_PF * N + l) * ls;
                pf_l2(Po + o + 3 * fs);
                pf_l2(Po + o + 4 * fs);
                if (SC) pf_l2(Po + o);
            }
        }
        double we[N], te[N], ro[N];
#pragma unroll
        for (int l = 1; l <= N; ++l) {
            const long long o = (long long)(k0 + l) * ls;
            we[l - 1] = Po[o + 3 * fs];
            te[l - 1] = Po[o + 4 * fs];
            ro[l - 1] = SC ? Po[o] : 0.0;
        }
#pragma unroll
        for (int l = N - 1; l >= 0; --l) {
            const int k = k0 + l;
            double s = 0.0;
            const double* Ur = LU + k * W + 2 * N;
#pragma unroll
            for (int j = 1; j <= 2 * N; ++j) s = fma(Ur[j], xw[l + j], s);
            xw[l] = (Y[k * T + tid] - s) * rU[k];
        }
        // extraction of levels k0+1 .. k0+N (element e now complete)
#pragma unroll
        for (int l = 1; l <= N; ++l) {
            const int k = k0 + l;
            double d = 0.0;
#pragma unroll
            for (int m = 0; m <= N; ++m) d = fma(sD[l * (N + 1) + m], xw[m], d);
            if (l == N && e + 1 < nez) {
                double d2 = 0.0;
#pragma unroll
                for (int m = 0; m <= N; ++m) d2 = fma(sD[m], xw[N + m], d2);
                d += d2;
            }
            extract(k, xw[l], d, ro[l - 1], we[l - 1], te[l - 1]);
        }
        if (e > 0) {
#pragma unroll
            for (int i = 2 * N; i >= 0; --i) xw[N + i] = xw[i];
        }
    }
    {   // bottom level: row 0 of element 0, boundary
        double d = 0.0;
#pragma unroll
        for (int m = 0; m <= N; ++m) d = fma(sD[m], xw[m], d);
        extract(0, xw[0], d, SC ? Po[0] : 0.0, Po[3 * fs], Po[4 * fs]);
    }
#undef TB
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
        if (!SC && a.pp_out) a.pp_out[loff(g, gx, gy, 0) + o] = solved_pprime(a, PT, M, k, rho, th);
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
