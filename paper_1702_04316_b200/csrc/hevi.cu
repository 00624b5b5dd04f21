// hevi.cu -- B200 (sm_100a) kernels and C ABI for the HEVI 1D-IMEX ARK2 step.
//
// Layout and schedule are described in DESIGN.md.  Short version:
//  * state lives on the unique-point lattice (one copy per DSS group), field
//    major, x fastest: the reference's cG E-vector state is bitwise
//    continuous (SURVEY finding 5), so the lattice holds the same numbers;
//  * the DSS of R(q) (euler.py:493, specgrid.py:535-540) is folded into the
//    derivatives: R is affine in the 18 gradient components with pointwise
//    coefficients, so the mass-weighted average of the per-copy R equals R
//    evaluated with mass-weighted averaged derivatives.  Each lattice point
//    reads its element lines and writes itself: no scatter, no atomics,
//    bit-stable, any partition gives the same bits;
//  * explicit kernel: one CTA per horizontal tile of element columns,
//    sweeping the element layers bottom-up through shared memory; the
//    element-face vertical derivative is carried in shared memory from the
//    layer below; ARK2 stage combinations fused into the epilogue;
//  * column kernel: one thread per vertical column, Schur RHS build,
//    banded forward/back substitution with the single shared LU factor
//    (box meshes: all columns identical), extraction -- fused.
#include "../../include/hevi.h"

// experiment builds: -DHEVI_DEV_N=4 instantiates one polynomial order only
// (every dispatch case maps to it; never used for the shipped library)
#ifdef HEVI_DEV_N
#define DN(n) HEVI_DEV_N
#else
#define DN(n) n
#endif
#ifndef HEVI_T44_TX
#define HEVI_T44_TX 4
#endif
#ifndef HEVI_T44_TY
#define HEVI_T44_TY 2
#endif
#ifndef HEVI_T44_MINB
#define HEVI_T44_MINB 1
#endif

#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

int fail(const char* what, cudaError_t e = cudaSuccess) {
    g_err = what;
    if (e != cudaSuccess) {
        g_err += ": ";
        g_err += cudaGetErrorString(e);
        return HEVI_ECUDA;
    }
    return HEVI_EARG;
}

#define CK(call)                                        \
    do {                                                \
        cudaError_t e_ = (call);                        \
        if (e_ != cudaSuccess) return fail(#call, e_);  \
    } while (0)

// ---------------------------------------------------------------------------
// parameter blocks (passed by value: live in the kernel constant bank)
// ---------------------------------------------------------------------------
struct Geo {
    int nex, ney, nez, X, Y, Z;
    int x0, y0, lX, lY, px;
    long long fs;
    int ex_b, ex_e, ey_b, ey_e;
    int slab;
};

struct Lev {
    const double *rho0, *theta0, *P0f, *drho0, *dth0, *G0, *H0, *F0z, *rho0G0;
    const double *E0, *c0, *irt0;   // EOS(rho0, theta0), E0 - P0f, 1/(rho0 theta0)
    const double *Th0, *iTh0, *F0c; // set2c: Theta0 = rho0 theta0, 1/Theta0, gamma P0f / Theta0
};

struct Phys {
    double g, R, P0, gamma;
};

enum { M_R = 0, M_L = 1, M_S1 = 2, M_S2 = 3, M_S3 = 4, M_RK = 5 };
// M_RK: one SSP RK(5,3) Shu-Osher stage (imexcore.py:111-126):
//   out = a_p * A + at_p * q + cb * R(q)     (A may be null: no a_p term)

struct EArgs {
    Geo g;
    Lev lv;
    Phys ph;
    const double *cx, *cy, *cz;
    const double *Dx, *Dy, *Dz;
    const double* q;
    double* out;   // M_R / M_L output, M_S3 new state
    double* P;     // predictor (fields 0,3,4)       [S1, S2]
    double* Quv;   // projected u,v of the stage      [S1 -> Q1, S2 -> A]
    double* A;     // S1 write, S2 read
    double* F;     // S1 write, S2 read/write, S3 read
    double dt, a_p, at_p, a_a, at_a, cb;
    unsigned* flags;
    int stage;
    double bc[16];   // binomial coefficients C(gamma, k), k = 1..15 (EOS series)
    int use_tma;     // 1: TMA staging (default); 0: cooperative loads
    int rk_final;    // M_RK: last stage (non-finite output check, imexcore.py:124-125)
    int af_tma;      // explicit_v2 M_S2/M_S3: A/F layer boxes by TMA (set by launch_e2)
    const double* pp_in;   // M_S2/M_S3 (set2nc): P' plane of the stage input from the column solve
    double* pp_out;        // explicit_col M_S3: P' plane of the new state (next step's stage 0)
    unsigned long long* dbg;   // HEVI_PHASE_TIMING builds: per-phase clock64 sums
    // tile subset of the column-sweep kernels (hevi_stage_ex HEVI_STAGE_*):
    // 0 every tile; 1 the interior rectangle [tb2, tb3) x [tb4, tb5); 2 the
    // ring of tiles around it (tb0 x tb1 tiles in all)
    int tmode;
    int tb[6];
};

struct SArgs {
    Geo g;
    Lev lv;
    Phys ph;
    const double* cz;
    const double* Dz;
    const double* LUb;     // M x (2nb-1)
    const double* lamtab;  // coefS | uA | den  (3*M)
    int nb;
    int ainv_identity;
    double lam;
    const double* P;       // predictor fields 0,3,4
    double* out;           // writes fields 0,3,4
    const double* src_uv;  // optional: copy u,v (with no-flux zeroing) from here
    double* pp_out;        // optional (set2nc): P' of the solved state, one lattice plane
    double bc[16];         // EOS series coefficients (as EArgs::bc)
};

__device__ __forceinline__ long long loff(const Geo& g, int gx, int gy, int gz) {
    return ((long long)gz * g.lY + (gy - g.y0)) * g.px + (gx - g.x0);
}

// position of lattice index `gi` on an axis with `ne` elements of order N:
// element line start (relative to the smem coordinate `l` of the point),
// derivative row, and whether the point is an element face shared with the
// element below/left (then row N of that element is added).
struct AxPt {
    int s0, row, s1;
    bool face;
};

__device__ __forceinline__ AxPt axpt(int gi, int l, int N, int ne) {
    AxPt r;
    if (gi == ne * N) {
        r.row = N;
        r.s0 = l - N;
        r.face = false;
        r.s1 = 0;
    } else {
        const int i = gi % N;
        r.row = i;
        r.s0 = l - i;
        r.face = (i == 0) && (gi > 0);
        r.s1 = l - N;
    }
    return r;
}

template <int N, int STRIDE>
__device__ __forceinline__ double dline(const double* s, const double* drow) {
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m <= N; ++m) acc = fma(drow[m], s[m * STRIDE], acc);
    return acc;
}

// ---------------------------------------------------------------------------
// explicit kernel: R(q) [+ L_V(q)] and the fused ARK2 stage epilogue
// ---------------------------------------------------------------------------
template <int NX, int NY, int NZ, int TX, int TY>
struct ETile {
    static constexpr int OX = TX * NX, OY = TY * NY;
    static constexpr int LX = OX + NX + 1, LY = OY + NY + 1, LZ = NZ + 1;
    static constexpr int PL = LX * LY, VOL = PL * LZ;
    static constexpr int CXW = OX + 1, CYW = OY + 1;
    static constexpr int NSF = 7;
    static constexpr int DXS = (NX + 1) * (NX + 1), DYS = (NY + 1) * (NY + 1),
                         DZS = (NZ + 1) * (NZ + 1);
    static constexpr size_t SMEM =
        sizeof(double) * (size_t)(NSF * VOL + NSF * CXW * CYW + DXS + DYS + DZS);
    static constexpr int PTS = OX * (OY + (NY == 1 ? 1 : 0)) * NZ;
    static constexpr int BLK0 = PTS < 64 ? 64 : (PTS > 512 ? 512 : PTS);
    static constexpr int BLK = (BLK0 + 31) / 32 * 32;
};

template <int NX, int NY, int NZ, int TX, int TY, int MODE>
__global__ void __launch_bounds__(ETile<NX, NY, NZ, TX, TY>::BLK)
    k_explicit(const EArgs a) {
    using T = ETile<NX, NY, NZ, TX, TY>;
    constexpr int LX = T::LX, PL = T::PL, VOL = T::VOL, CXW = T::CXW, CYW = T::CYW;
    constexpr int BLK = T::BLK;
    constexpr bool NEED_L = (MODE == M_L || MODE == M_S1 || MODE == M_S2);
    constexpr bool NEED_R = (MODE != M_L);
    extern __shared__ __align__(16) double sm[];
    double* S = sm;
    double* Cr = S + T::NSF * VOL;
    double* sDx = Cr + T::NSF * CXW * CYW;
    double* sDy = sDx + T::DXS;
    double* sDz = sDy + T::DYS;

    const Geo& g = a.g;
    const int tid = threadIdx.x;
    const int ex0 = g.ex_b + blockIdx.x * TX;
    const int ey0 = g.ey_b + blockIdx.y * TY;
    const int nxe = min(TX, g.ex_e - ex0);
    const int nye = min(TY, g.ey_e - ey0);
    const int oxn = nxe * NX + ((ex0 + nxe == g.nex) ? 1 : 0);
    const int oyn = nye * NY + ((ey0 + nye == g.ney) ? 1 : 0);
    const int gxlo = (ex0 - 1) * NX, gylo = (ey0 - 1) * NY;
    const double gr = a.ph.g;

    for (int i = tid; i < T::DXS; i += BLK) sDx[i] = a.Dx[i];
    for (int i = tid; i < T::DYS; i += BLK) sDy[i] = a.Dy[i];
    for (int i = tid; i < T::DZS; i += BLK) sDz[i] = a.Dz[i];

    for (int ez = 0; ez < g.nez; ++ez) {
        const int gz0 = ez * NZ;
        // ---------------- load the element layer (+ low-side halo) --------
        for (int idx = tid; idx < VOL; idx += BLK) {
            const int lx = idx % LX;
            const int t = idx / LX;
            const int ly = t % T::LY;
            const int lz = t / T::LY;
            const int gx = gxlo + lx, gy = gylo + ly, gz = gz0 + lz;
            const int ix = gx - g.x0, iy = gy - g.y0;
            double r = 0.0, u = 0.0, v = 0.0, w = 0.0, th = 0.0, pp = 0.0, pl = 0.0;
            if (gx >= 0 && gx < g.X && gy >= 0 && gy < g.Y && ix >= 0 && ix < g.lX && iy >= 0 &&
                iy < g.lY) {
                const double* qp = a.q + ((long long)gz * g.lY + iy) * g.px + ix;
                r = __ldg(qp);
                u = __ldg(qp + g.fs);
                v = __ldg(qp + 2 * g.fs);
                w = __ldg(qp + 3 * g.fs);
                th = __ldg(qp + 4 * g.fs);
                if (NEED_R) {
                    // euler.py:454-457 and equation_of_state (euler.py:185)
                    const double rho = __ldg(a.lv.rho0 + gz) + r;
                    const double theta = __ldg(a.lv.theta0 + gz) + th;
                    pp = a.ph.P0 * pow(rho * a.ph.R * theta / a.ph.P0, a.ph.gamma) -
                         __ldg(a.lv.P0f + gz);
                }
                if (NEED_L) pl = __ldg(a.lv.G0 + gz) * r + __ldg(a.lv.H0 + gz) * th;
            }
            S[0 * VOL + idx] = r;
            S[1 * VOL + idx] = u;
            S[2 * VOL + idx] = v;
            S[3 * VOL + idx] = w;
            S[4 * VOL + idx] = th;
            S[5 * VOL + idx] = pp;
            S[6 * VOL + idx] = pl;
        }
        __syncthreads();
        // ---------------- per owned point ---------------------------------
        const int ozn = NZ + ((ez == g.nez - 1) ? 1 : 0);
        const int npts = oxn * oyn * ozn;
        for (int p = tid; p < npts; p += BLK) {
            const int ox = p % oxn;
            const int t = p / oxn;
            const int oy = t % oyn;
            const int oz = t / oyn;
            const int gx = ex0 * NX + ox, gy = ey0 * NY + oy, gz = gz0 + oz;
            const int lx = ox + NX, ly = oy + NY, lz = oz;
            const AxPt ax = axpt(gx, lx, NX, g.nex);
            const AxPt ay = axpt(gy, ly, NY, g.ney);
            const AxPt az = axpt(gz, lz, NZ, g.nez);
            const double cx = __ldg(a.cx + gx), cy = __ldg(a.cy + gy), cz = __ldg(a.cz + gz);
            double dxa[NX + 1], dxb[NX + 1], dya[NY + 1], dyb[NY + 1], dza[NZ + 1];
#pragma unroll
            for (int m = 0; m <= NX; ++m) {
                dxa[m] = sDx[ax.row * (NX + 1) + m];
                dxb[m] = sDx[NX * (NX + 1) + m];
            }
#pragma unroll
            for (int m = 0; m <= NY; ++m) {
                dya[m] = sDy[ay.row * (NY + 1) + m];
                dyb[m] = sDy[NY * (NY + 1) + m];
            }
#pragma unroll
            for (int m = 0; m <= NZ; ++m) dza[m] = sDz[az.row * (NZ + 1) + m];
            const int cidx = oy * CXW + ox;
            const bool zface = az.face;

            double dX[6], dY[6], dZ[7];
#pragma unroll
            for (int f = 0; f < 6; ++f) {
                const double* sx = S + f * VOL + lz * PL + ly * LX;
                double d = dline<NX, 1>(sx + ax.s0, dxa);
                if (ax.face) d += dline<NX, 1>(sx + ax.s1, dxb);
                dX[f] = cx * d;
                const double* sy = S + f * VOL + lz * PL + lx;
                double e = dline<NY, LX>(sy + ay.s0 * LX, dya);
                if (ay.face) e += dline<NY, LX>(sy + ay.s1 * LX, dyb);
                dY[f] = cy * e;
            }
#pragma unroll
            for (int f = 0; f < 7; ++f) {
                if (f == 6 && !NEED_L) {
                    dZ[6] = 0.0;
                    continue;
                }
                if (f == 5 && !NEED_R) {
                    dZ[5] = 0.0;
                    continue;
                }
                const double* sz = S + f * VOL + ly * LX + lx;
                double d = dline<NZ, PL>(sz + az.s0 * PL, dza);
                if (zface) d += Cr[f * CXW * CYW + cidx];
                dZ[f] = cz * d;
            }
            // partial (row N) of this element layer at its top face, consumed by
            // the face level of the next layer
            if (oz == 0 && ez + 1 < g.nez) {
                double dzn[NZ + 1];
#pragma unroll
                for (int m = 0; m <= NZ; ++m) dzn[m] = sDz[NZ * (NZ + 1) + m];
#pragma unroll
                for (int f = 0; f < 7; ++f) {
                    const double* sz = S + f * VOL + ly * LX + lx;
                    Cr[f * CXW * CYW + cidx] = dline<NZ, PL>(sz, dzn);
                }
            }

            const int c0 = lz * PL + ly * LX + lx;
            const double r = S[0 * VOL + c0], u = S[1 * VOL + c0], v = S[2 * VOL + c0],
                         w = S[3 * VOL + c0], th = S[4 * VOL + c0];
            const double rho0 = __ldg(a.lv.rho0 + gz);
            const double drho0 = __ldg(a.lv.drho0 + gz);
            const double dth0 = __ldg(a.lv.dth0 + gz);
            const bool bx = (gx == 0) || (gx == g.X - 1);
            const bool by = g.slab || (gy == 0) || (gy == g.Y - 1);
            const bool bz = (gz == 0) || (gz == g.Z - 1);

            double R0 = 0.0, R1 = 0.0, R2 = 0.0, R3 = 0.0, R4 = 0.0;
            if (NEED_R) {
                const double rho = rho0 + r;
                const double theta = __ldg(a.lv.theta0 + gz) + th;
                const bool finite = isfinite(r) && isfinite(u) && isfinite(v) && isfinite(w) &&
                                    isfinite(th);
                if (!finite) atomicOr(a.flags, HEVI_F_NONFINITE_IN(a.stage));
                if (!(rho > 0.0) || !(theta > 0.0)) atomicOr(a.flags, HEVI_F_EOS(a.stage));
                // euler.nonlinear_rhs set2nc (euler.py:458-473), DSS folded into dX/dY/dZ
                const double divu = (dX[1] + dY[2]) + dZ[3];
                const double rinv = 1.0 / rho;
                R0 = -(((u * dX[0] + v * dY[0]) + w * dZ[0]) + w * drho0 + rho * divu);
                R1 = -(((u * dX[1] + v * dY[1]) + w * dZ[1]) + dX[5] * rinv);
                R2 = -(((u * dX[2] + v * dY[2]) + w * dZ[2]) + dY[5] * rinv);
                R3 = -(((u * dX[3] + v * dY[3]) + w * dZ[3]) + dZ[5] * rinv + (r * rinv) * gr);
                R4 = -(((u * dX[4] + v * dY[4]) + w * dZ[4]) + w * dth0);
                // euler.zero_normal_velocity after the DSS (euler.py:494-496)
                if (bx) R1 = 0.0;
                if (by) R2 = 0.0;
                if (bz) R3 = 0.0;
            }
            double L0 = 0.0, L3 = 0.0, L4 = 0.0;
            if (NEED_L) {
                // euler.linear_operator(vertical_only=True), set2nc (euler.py:333-361)
                L0 = -(w * drho0 + rho0 * dZ[3]);
                L3 = bz ? 0.0 : -(dZ[6] / rho0 + (r / rho0) * gr);
                L4 = -(w * dth0);
            }
            const long long o = loff(g, gx, gy, gz);
            const long long fs = g.fs;
            if (MODE == M_R) {
                a.out[o] = R0;
                a.out[o + fs] = R1;
                a.out[o + 2 * fs] = R2;
                a.out[o + 3 * fs] = R3;
                a.out[o + 4 * fs] = R4;
            } else if (MODE == M_L) {
                a.out[o] = L0;
                a.out[o + fs] = 0.0;
                a.out[o + 2 * fs] = 0.0;
                a.out[o + 3 * fs] = L3;
                a.out[o + 4 * fs] = L4;
            } else if (MODE == M_S1) {
                // imexcore.ark_imex_step (imexcore.py:398-403, 409-411)
                const double dt = a.dt;
                const double qv[5] = {r, u, v, w, th};
                const double Rv[5] = {R0, R1, R2, R3, R4};
                const double Lv[5] = {L0, 0.0, 0.0, L3, L4};
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
                const double Rv[5] = {R0, R1, R2, R3, R4};
                const double Lv[5] = {L0, 0.0, 0.0, L3, L4};
                double pr[5];
#pragma unroll
                for (int f = 0; f < 5; ++f) {
                    const double acc = a.A[o + f * fs];
                    pr[f] = acc + dt * (a.a_p * (Rv[f] - Lv[f]) + a.at_p * Lv[f]);
                    a.F[o + f * fs] = a.F[o + f * fs] + a.cb * Rv[f];
                }
                a.P[o] = pr[0];
                a.P[o + 3 * fs] = pr[3];
                a.P[o + 4 * fs] = pr[4];
                a.Quv[o + fs] = bx ? 0.0 : pr[1];
                a.Quv[o + 2 * fs] = by ? 0.0 : pr[2];
            } else if (MODE == M_RK) {
                const double Rv[5] = {R0, R1, R2, R3, R4};
                const double qv[5] = {r, u, v, w, th};
                bool fin = true;
#pragma unroll
                for (int f = 0; f < 5; ++f) {
                    double val = a.A ? a.a_p * a.A[o + f * fs] : 0.0;
                    val = val + a.at_p * qv[f];
                    val = val + a.cb * Rv[f];
                    fin = fin && isfinite(val);
                    a.out[o + f * fs] = val;
                }
                if (a.rk_final && !fin) atomicOr(a.flags, HEVI_F_NONFINITE_OUT);
            } else {  // M_S3
                const double Rv[5] = {R0, R1, R2, R3, R4};
                bool fin = true;
#pragma unroll
                for (int f = 0; f < 5; ++f) {
                    const double val = a.F[o + f * fs] + a.cb * Rv[f];
                    fin = fin && isfinite(val);
                    a.out[o + f * fs] = val;
                }
                if (!fin) atomicOr(a.flags, HEVI_F_NONFINITE_OUT);
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// column kernel: Schur RHS -> banded substitution -> extraction (one thread
// per vertical column; imexcore.py:229-243, columnsolve.py:156-181,
// imexcore.py:273-287)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void lev_elem(int k, int N, int ne, int& s0, int& row, bool& face) {
    if (k == ne * N) {
        row = N;
        s0 = k - N;
        face = false;
    } else {
        row = k % N;
        s0 = k - row;
        face = (row == 0) && (k > 0);
    }
}

template <int NZ>
__device__ __forceinline__ double col_deriv(const double* buf, int T, int tid, int k, int nez,
                                            const double* sD, double c) {
    int s0, row;
    bool face;
    lev_elem(k, NZ, nez, s0, row, face);
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m <= NZ; ++m) acc = fma(sD[row * (NZ + 1) + m], buf[(s0 + m) * T + tid], acc);
    if (face) {
        double acc2 = 0.0;
#pragma unroll
        for (int m = 0; m <= NZ; ++m)
            acc2 = fma(sD[NZ * (NZ + 1) + m], buf[(k - NZ + m) * T + tid], acc2);
        acc += acc2;
    }
    return c * acc;
}

template <int NZ>
__global__ void k_solve(const SArgs a) {
    extern __shared__ __align__(16) double sm[];
    const Geo& g = a.g;
    const int M = g.Z;
    const int T = blockDim.x;
    const int tid = threadIdx.x;
    const int W = 2 * a.nb - 1;
    double* tG0 = sm;
    double* tH0 = tG0 + M;
    double* trho0 = tH0 + M;
    double* tF0z = trho0 + M;
    double* trG = tF0z + M;
    double* tdth0 = trG + M;
    double* tcz = tdth0 + M;
    double* tcoef = tcz + M;
    double* tuA = tcoef + M;
    double* tden = tuA + M;
    double* LU = tden + M;
    double* sD = LU + M * W;
    double* U = sD + (NZ + 1) * (NZ + 1);
    double* Yb = U + M * T;
    for (int k = tid; k < M; k += T) {
        tG0[k] = a.lv.G0[k];
        tH0[k] = a.lv.H0[k];
        trho0[k] = a.lv.rho0[k];
        tF0z[k] = a.lv.F0z[k];
        trG[k] = a.lv.rho0G0[k];
        tdth0[k] = a.lv.dth0[k];
        tcz[k] = a.cz[k];
        tcoef[k] = a.lamtab[k];
        tuA[k] = a.lamtab[M + k];
        tden[k] = a.lamtab[2 * M + k];
    }
    for (int i = tid; i < M * W; i += T) LU[i] = a.LUb[i];
    for (int i = tid; i < (NZ + 1) * (NZ + 1); i += T) sD[i] = a.Dz[i];
    __syncthreads();

    // owned columns
    const int xlo = g.ex_b * NZ;  // N (horizontal) == NZ for both layouts
    const int cntx = (g.ex_e - g.ex_b) * NZ + (g.ex_e == g.nex ? 1 : 0);
    const int NYo = g.slab ? 1 : NZ;
    const int ylo = g.ey_b * NYo;
    const int cnty = (g.ey_e - g.ey_b) * NYo + (g.ey_e == g.ney ? 1 : 0);
    const int c = blockIdx.x * T + tid;
    if (c >= cntx * cnty) return;
    const int gx = xlo + c % cntx;
    const int gy = ylo + c / cntx;
    const int gys = g.slab ? 0 : gy;  // slab: columns keyed by x only
    const long long fs = g.fs;
    const double lam = a.lam, gr = a.ph.g;
    const bool ident = a.ainv_identity != 0;
    const int nez = g.nez;

    // pass 1: ua_z (imexcore.py:236-241) of the source column
    for (int k = 0; k < M; ++k) {
        const long long o = loff(g, gx, gys, k);
        const double we = a.P[o + 3 * fs], te = a.P[o + 4 * fs];
        double v = we + (tcoef[k] * te) * gr;
        if (!ident) v = v - tuA[k] * ((tdth0[k] * v) / tden[k]);
        U[k * T + tid] = (k == 0 || k == M - 1) ? 0.0 : v;
    }
    // pass 2: rhs = Pe - lam (F0 . ua + rho0 G0 div_vc ua), forward substitution
    const int nb = a.nb;
    for (int k = 0; k < M; ++k) {
        const long long o = loff(g, gx, gys, k);
        const double re = a.P[o], te = a.P[o + 4 * fs];
        const double ua = U[k * T + tid];
        const double dua = col_deriv<NZ>(U, T, tid, k, nez, sD, tcz[k]);
        const double Pe = tG0[k] * re + tH0[k] * te;
        const double rhs = Pe - lam * (tF0z[k] * ua + trG[k] * dua);
        double s = 0.0;
        const int j0 = max(0, k - nb + 1);
        for (int j = j0; j < k; ++j) s = fma(LU[k * W + (j - k + nb - 1)], Yb[j * T + tid], s);
        Yb[k * T + tid] = rhs - s;
    }
    // pass 3: back substitution
    for (int k = M - 1; k >= 0; --k) {
        double s = 0.0;
        const int j1 = min(k + nb, M);
        for (int j = k + 1; j < j1; ++j) s = fma(LU[k * W + (j - k + nb - 1)], Yb[j * T + tid], s);
        Yb[k * T + tid] = (Yb[k * T + tid] - s) / LU[k * W + (nb - 1)];
    }
    // pass 4: extraction (imexcore.py:277-287) on the own column
    for (int k = 0; k < M; ++k) {
        const long long o = loff(g, gx, gy, k);
        const double we = a.P[o + 3 * fs], te = a.P[o + 4 * fs];
        const double Pk = Yb[k * T + tid];
        const double dP = col_deriv<NZ>(Yb, T, tid, k, nez, sD, tcz[k]);
        const bool bz = (k == 0) || (k == M - 1);
        double ua = we + (tcoef[k] * te) * gr;
        double up = lam * (dP / trho0[k] + (Pk / (tG0[k] * trho0[k])) * gr);
        if (!ident) {
            ua = ua - tuA[k] * ((tdth0[k] * ua) / tden[k]);
            up = up - tuA[k] * ((tdth0[k] * up) / tden[k]);
        }
        if (bz) {
            ua = 0.0;
            up = 0.0;
        }
        const double w = ua - up;
        const double th = te - lam * (w * tdth0[k]);
        const double rho = (Pk - tH0[k] * th) / tG0[k];
        a.out[o] = rho;
        a.out[o + 3 * fs] = w;
        a.out[o + 4 * fs] = th;
        if (a.src_uv) {
            const bool bx = (gx == 0) || (gx == g.X - 1);
            const bool by = g.slab || (gy == 0) || (gy == g.Y - 1);
            a.out[o + fs] = bx ? 0.0 : a.src_uv[o + fs];
            a.out[o + 2 * fs] = by ? 0.0 : a.src_uv[o + 2 * fs];
        }
    }
}

// ---------------------------------------------------------------------------
// factorization (setup, once per lam): per-level lam tables, probing of the
// Schur column operator (columnsolve.py:75-108 on one column), no-pivot
// banded LU (columnsolve.py:111-138)
// ---------------------------------------------------------------------------
struct FArgs {
    Lev lv;
    double g, lam;
    const double* cz;
    const double* Dz;
    int N, nez, M, ainv_identity, eqset;
    double* lamtab;  // coefS | uA | den
    double* vtab;    // V_NT x M tables of the v2 column kernel
    double* A;       // M*M dense, row-major, zeroed
    unsigned* flags;
};

__global__ void k_lamtab(const FArgs a) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= a.M) return;
    const double lam = a.lam;
    // imexcore.py:236  coef = lam * H0 / (G0 * rho0)
    a.lamtab[k] = lam * a.lv.H0[k] / (a.lv.G0[k] * a.lv.rho0[k]);
    // imexcore.py:207-213  u = lam^2/theta0 * g;  den = 1 + w . u
    const double uA = (lam * lam / a.lv.theta0[k]) * a.g;
    const double den = 1.0 + a.lv.dth0[k] * uA;
    a.lamtab[a.M + k] = uA;
    a.lamtab[2 * a.M + k] = den;
    if (!a.ainv_identity && fabs(den) < 1e-12) atomicOr(a.flags, HEVI_F_AINV);
    const int M = a.M;
    double* t = a.vtab;
    t[0 * M + k] = a.lv.G0[k];
    t[1 * M + k] = a.lv.H0[k];
    t[2 * M + k] = a.lv.F0z[k];
    t[3 * M + k] = a.lv.rho0G0[k];
    t[4 * M + k] = a.cz[k];
    t[5 * M + k] = a.lamtab[k];
    t[6 * M + k] = uA;
    t[7 * M + k] = den;
    t[8 * M + k] = a.lv.dth0[k];
    t[9 * M + k] = 1.0 / a.lv.rho0[k];
    t[10 * M + k] = 1.0 / (a.lv.G0[k] * a.lv.rho0[k]);
    t[11 * M + k] = 1.0 / a.lv.G0[k];
    // set2c (imexcore.py:239-240, 254-255, 266-268, 288-297): G0 = theta0
    t[12 * M + k] = a.lv.F0c[k];
    t[13 * M + k] = a.lv.theta0[k];
    t[14 * M + k] = 1.0 / (a.lv.F0c[k] * a.lv.theta0[k]);
    t[15 * M + k] = 1.0 / a.lv.theta0[k];
}

__device__ double f_unit(int l, int j) { return l == j ? 1.0 : 0.0; }

// column j of A = lhs_schur(e_j)
__global__ void k_probe(const FArgs a) {
    const int N = a.N, M = a.M, nez = a.nez;
    const double lam = a.lam, gr = a.g;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < M; j += gridDim.x * blockDim.x) {
        double up[2 * 16 + 1];  // levels j-N .. j+N (N <= 16)
        for (int t = 0; t <= 2 * N; ++t) {
            const int k = j - N + t;
            up[t] = 0.0;
            if (k < 0 || k >= M) continue;
            int s0, row;
            bool face;
            lev_elem(k, N, nez, s0, row, face);
            double acc = 0.0;
            for (int m = 0; m <= N; ++m) acc = fma(a.Dz[row * (N + 1) + m], f_unit(s0 + m, j), acc);
            if (face) {
                double acc2 = 0.0;
                for (int m = 0; m <= N; ++m)
                    acc2 = fma(a.Dz[N * (N + 1) + m], f_unit(k - N + m, j), acc2);
                acc += acc2;
            }
            const double dP = a.cz[k] * acc;
            // imexcore._up (imexcore.py:250-255)
            double v = a.eqset == 0
                           ? lam * (dP / a.lv.rho0[k] + (f_unit(k, j) / (a.lv.G0[k] * a.lv.rho0[k])) * gr)
                           : lam * (dP + (f_unit(k, j) / (a.lv.F0c[k] * a.lv.theta0[k])) * gr);
            if (!a.ainv_identity) {
                const double uA = a.lamtab[M + k], den = a.lamtab[2 * M + k];
                v = v - uA * ((a.lv.dth0[k] * v) / den);
            }
            up[t] = (k == 0 || k == M - 1) ? 0.0 : v;
        }
        for (int k = max(0, j - 2 * N); k <= min(M - 1, j + 2 * N); ++k) {
            int s0, row;
            bool face;
            lev_elem(k, N, nez, s0, row, face);
            auto upv = [&](int l) -> double {
                const int t = l - (j - N);
                return (t >= 0 && t <= 2 * N) ? up[t] : 0.0;
            };
            double acc = 0.0;
            for (int m = 0; m <= N; ++m) acc = fma(a.Dz[row * (N + 1) + m], upv(s0 + m), acc);
            if (face) {
                double acc2 = 0.0;
                for (int m = 0; m <= N; ++m) acc2 = fma(a.Dz[N * (N + 1) + m], upv(k - N + m), acc2);
                acc += acc2;
            }
            const double dup = a.cz[k] * acc;
            // imexcore._helmholtz_flux (imexcore.py:263-268), lhs_schur (:270-271)
            const double helm =
                a.eqset == 0 ? lam * (a.lv.F0z[k] * upv(k) + a.lv.rho0G0[k] * dup)
                             : a.lv.F0c[k] * lam * (a.lv.theta0[k] * dup + a.lv.dth0[k] * upv(k));
            a.A[(long long)k * M + j] = f_unit(k, j) - helm;
        }
    }
}

// single-CTA dense LU restricted to the band, band detection and packing
__global__ void k_lu_dense(double* A, double* LU, double* LUb, int M, int* nb_out,
                           unsigned* flags, int N2, double* LU2, double* rU) {
    __shared__ double red[1024];
    __shared__ int redi[1024];
    __shared__ double s_norm;
    __shared__ int s_nb;
    const int tid = threadIdx.x, T = blockDim.x;
    double mx = 0.0;
    for (int i = tid; i < M * M; i += T) mx = fmax(mx, fabs(A[i]));
    red[tid] = mx;
    __syncthreads();
    for (int s = T / 2; s > 0; s >>= 1) {
        if (tid < s) red[tid] = fmax(red[tid], red[tid + s]);
        __syncthreads();
    }
    if (tid == 0) s_norm = red[0];
    __syncthreads();
    const double norm = s_norm;
    // bandwidth from the sparsity pattern (columnsolve.py:103-106)
    int bw = -1;
    for (int i = tid; i < M * M; i += T) {
        if (fabs(A[i]) > 1e-14 * norm) bw = max(bw, abs(i / M - i % M));
    }
    redi[tid] = bw;
    __syncthreads();
    for (int s = T / 2; s > 0; s >>= 1) {
        if (tid < s) redi[tid] = max(redi[tid], redi[tid + s]);
        __syncthreads();
    }
    if (tid == 0) s_nb = redi[0] + 1;
    __syncthreads();
    const int nb = s_nb < 1 ? 1 : s_nb;
    for (int i = tid; i < M * M; i += T) LU[i] = A[i];
    __syncthreads();
    for (int k = 0; k < M; ++k) {
        double piv = LU[k * M + k];
        if (fabs(piv) < 1e-12 * norm) {
            if (tid == 0) atomicOr(flags, 1u);   // degenerate: the plan falls back to pivoted LU
            piv = 1.0;
        }
        const int E = min(k + nb, M);
        for (int r = k + 1 + tid; r < E; r += T) LU[r * M + k] /= piv;
        __syncthreads();
        const int n = E - (k + 1);
        for (int t = tid; t < n * n; t += T) {
            const int r = k + 1 + t / n, cc = k + 1 + t % n;
            LU[r * M + cc] -= LU[r * M + k] * LU[k * M + cc];
        }
        __syncthreads();
    }
    const int W = 2 * nb - 1;
    for (int i = tid; i < M * W; i += T) {
        const int k = i / W, d = i % W;
        const int j = k + d - (nb - 1);
        LUb[i] = (j >= 0 && j < M) ? LU[k * M + j] : 0.0;
    }
    const int W2 = 4 * N2 + 1;
    for (int i = tid; i < M * W2; i += T) {
        const int k = i / W2, d = i % W2;
        const int j = k + d - 2 * N2;
        LU2[i] = (j >= 0 && j < M && abs(j - k) < nb) ? LU[k * M + j] : 0.0;
    }
    for (int k = tid; k < M; k += T) rU[k] = 1.0 / LU[k * M + k];
    if (tid == 0) *nb_out = nb;
}

// Partial-pivoting dense LU of one M x M row-major matrix, in place, by one
// CTA: the pivoted fallback of columnsolve.factor_with_fallback
// (columnsolve.py:141-153; scipy.linalg.lu_factor = LAPACK getrf semantics:
// piv[k] = row interchanged with row k, first max |a_ik| wins, an exactly
// zero pivot is reported through *info = k+1 and its column is not scaled).
__device__ void lu_pivot_cta(double* LU, int* piv, int M, int* info) {
    __shared__ double rv[256];
    __shared__ int ri[256];
    __shared__ int s_p;
    const int tid = threadIdx.x, T = blockDim.x;
    if (tid == 0 && info) *info = 0;
    for (int k = 0; k < M; ++k) {
        double best = -1.0;
        int bi = M;
        for (int r = k + tid; r < M; r += T) {
            const double v = fabs(LU[r * M + k]);
            if (v > best || (v == best && r < bi)) { best = v; bi = r; }
        }
        rv[tid] = best;
        ri[tid] = bi;
        __syncthreads();
        for (int s = T / 2; s > 0; s >>= 1) {
            if (tid < s) {
                const double v = rv[tid + s];
                const int i = ri[tid + s];
                if (v > rv[tid] || (v == rv[tid] && i < ri[tid])) { rv[tid] = v; ri[tid] = i; }
            }
            __syncthreads();
        }
        if (tid == 0) {
            s_p = ri[0];
            piv[k] = ri[0];
            if (rv[0] == 0.0 && info && *info == 0) *info = k + 1;
        }
        __syncthreads();
        const int p = s_p;
        if (p != k)
            for (int c = tid; c < M; c += T) {
                const double t = LU[k * M + c];
                LU[k * M + c] = LU[p * M + c];
                LU[p * M + c] = t;
            }
        __syncthreads();
        const double pv = LU[k * M + k];
        if (pv != 0.0)
            for (int r = k + 1 + tid; r < M; r += T) LU[r * M + k] /= pv;
        __syncthreads();
        const int n = M - (k + 1);
        for (int t = tid; t < n * n; t += T) {
            const int r = k + 1 + t / n, c = k + 1 + t % n;
            LU[r * M + c] -= LU[r * M + k] * LU[k * M + c];
        }
        __syncthreads();
    }
}

// plan factor fallback: LUP = pivoted LU of the shared column matrix A
__global__ void k_lu_pivot(const double* A, double* LUP, int* piv, int M, int* info) {
    for (int i = threadIdx.x; i < M * M; i += blockDim.x) LUP[i] = A[i];
    __syncthreads();
    lu_pivot_cta(LUP, piv, M, info);
}

// batched API (columnsolve.factor_with_fallback): one CTA per column
__global__ void k_lu_pivot_batched(double* A, int* piv, int M, int* info) {
    const long long c = blockIdx.x;
    lu_pivot_cta(A + c * M * M, piv + c * M, M, info + c);
}

// batched pivoted substitution (scipy.linalg.lu_solve): one thread per column
__global__ void k_lu_pivot_solve(const double* LU, const int* piv, double* x, int n_col, int M) {
    const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_col) return;
    const double* A = LU + c * M * M;
    const int* pv = piv + c * M;
    double* b = x + c * M;
    for (int i = 0; i < M; ++i) {
        const int p = pv[i];
        if (p != i) {
            const double t = b[i];
            b[i] = b[p];
            b[p] = t;
        }
    }
    for (int i = 1; i < M; ++i) {
        double s = 0.0;
        for (int j = 0; j < i; ++j) s = fma(A[i * M + j], b[j], s);
        b[i] -= s;
    }
    for (int i = M - 1; i >= 0; --i) {
        double s = 0.0;
        for (int j = i + 1; j < M; ++j) s = fma(A[i * M + j], b[j], s);
        b[i] = (b[i] - s) / A[i * M + i];
    }
}

// ---------------------------------------------------------------------------
// Run diagnostics (bench.total_mass / max_perturbations, bench.py:131-137) on
// the lattice: mass = sum_g Wx Wy Wz (rho0 + rho'), max |rho'|, max |q4|.
// Fixed grid and reduction order, so the result is bitwise reproducible.
// ---------------------------------------------------------------------------
constexpr int DIAG_BLOCKS = 592, DIAG_T = 256;

__global__ void k_diag_partial(Geo g, const double* __restrict__ q, const double* __restrict__ rho0,
                               const double* __restrict__ wx, const double* __restrict__ wy,
                               const double* __restrict__ wz, double* part) {
    __shared__ double sm[3][DIAG_T];
    const long long n = (long long)g.Z * g.lY * g.lX;
    double m = 0.0, mr = 0.0, mt = 0.0;
    for (long long i = (long long)blockIdx.x * DIAG_T + threadIdx.x; i < n;
         i += (long long)DIAG_BLOCKS * DIAG_T) {
        const int x = (int)(i % g.lX);
        const long long t = i / g.lX;
        const int y = (int)(t % g.lY);
        const int z = (int)(t / g.lY);
        const long long o = ((long long)z * g.lY + y) * g.px + x;
        const double r = q[o], th = q[o + 4 * g.fs];
        m = fma(wz[z] * wy[y + g.y0] * wx[x + g.x0], rho0[z] + r, m);
        mr = fmax(mr, fabs(r));
        mt = fmax(mt, fabs(th));
    }
    sm[0][threadIdx.x] = m;
    sm[1][threadIdx.x] = mr;
    sm[2][threadIdx.x] = mt;
    __syncthreads();
    for (int s = DIAG_T / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            sm[0][threadIdx.x] += sm[0][threadIdx.x + s];
            sm[1][threadIdx.x] = fmax(sm[1][threadIdx.x], sm[1][threadIdx.x + s]);
            sm[2][threadIdx.x] = fmax(sm[2][threadIdx.x], sm[2][threadIdx.x + s]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[blockIdx.x] = sm[0][0];
        part[DIAG_BLOCKS + blockIdx.x] = sm[1][0];
        part[2 * DIAG_BLOCKS + blockIdx.x] = sm[2][0];
    }
}

__global__ void k_diag_final(const double* part, double* out) {
    if (threadIdx.x != 0) return;
    double m = 0.0, mr = 0.0, mt = 0.0;
    for (int b = 0; b < DIAG_BLOCKS; ++b) {
        m += part[b];
        mr = fmax(mr, part[DIAG_BLOCKS + b]);
        mt = fmax(mt, part[2 * DIAG_BLOCKS + b]);
    }
    out[0] = m;
    out[1] = mr;
    out[2] = mt;
}

// ---------------------------------------------------------------------------
// E-vector <-> lattice
// ---------------------------------------------------------------------------
struct CArgs {
    Geo g;
    int N, Ny;
    long long nel;
};

__device__ __forceinline__ void rep_of(int gi, int N, int ne, int& k, int& i) {
    // first occurrence in flat element order: the lower element on a face
    if (gi > 0 && gi % N == 0) {
        k = gi / N - 1;
        i = N;
    } else {
        k = min(gi / N, ne - 1);
        i = gi - k * N;
    }
}

__global__ void k_e2l(const double* E, double* Lt, const CArgs a, int nf) {
    const Geo& g = a.g;
    const long long n = (long long)g.lX * g.lY * g.Z;
    const int nr = a.N + 1, ns = a.Ny + 1, nt = a.N + 1;
    const long long npe = (long long)nr * ns * nt;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        const int ix = idx % g.lX;
        const long long t = idx / g.lX;
        const int iy = t % g.lY;
        const int gz = t / g.lY;
        const int gx = g.x0 + ix, gy = g.y0 + iy;
        int kx, i, ky, j, kz, k;
        rep_of(gx, a.N, g.nex, kx, i);
        rep_of(gy, a.Ny, g.ney, ky, j);
        rep_of(gz, a.N, g.nez, kz, k);
        const long long e = ((long long)kz * g.ney + ky) * g.nex + kx;
        const long long node = e * npe + ((long long)k * ns + j) * nr + i;
        const long long o = ((long long)gz * g.lY + iy) * g.px + ix;
        for (int f = 0; f < nf; ++f) Lt[f * g.fs + o] = E[f * a.nel * npe + node];
    }
}

__global__ void k_l2e(const double* Lt, double* E, const CArgs a, int nf) {
    const Geo& g = a.g;
    const int nr = a.N + 1, ns = a.Ny + 1, nt = a.N + 1;
    const long long npe = (long long)nr * ns * nt;
    const long long n = a.nel * npe;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = idx % nr;
        long long t = idx / nr;
        const int j = t % ns;
        t /= ns;
        const int k = t % nt;
        const long long e = t / nt;
        const int kx = e % g.nex;
        const int ky = (e / g.nex) % g.ney;
        const int kz = e / ((long long)g.nex * g.ney);
        const int gx = kx * a.N + i, gy = ky * a.Ny + j, gz = kz * a.N + k;
        const long long o = ((long long)gz * g.lY + (gy - g.y0)) * g.px + (gx - g.x0);
        for (int f = 0; f < nf; ++f) E[f * n + idx] = Lt[f * g.fs + o];
    }
}

// specgrid.apply_dss (specgrid.py:535-540) on E-vectors: every coincident
// copy of a lattice point takes the mass-weighted average of all copies,
// sum_c w_c f_c / sum_c w_c, summed in the reference's flat node order
// (elements in (kz, ky, kx) order, the lower element first on a face).
// w_c = Wx[kx][i] Wy[ky][j] Wz[kz][k] (quadrature weight x half element
// width per axis: the box mesh's wJ).  One thread per lattice point, no
// atomics; any discontinuous E-vector is accepted.
__global__ void k_dss(const double* __restrict__ Ein, double* __restrict__ Eout, const CArgs a, int nf,
                      const double* __restrict__ Wx, const double* __restrict__ Wy,
                      const double* __restrict__ Wz) {
    const Geo& g = a.g;
    const int X = g.X, Y = g.Y, Zl = g.Z;
    const long long n = (long long)X * Y * Zl;
    const int nr = a.N + 1, ns = a.Ny + 1, nt = a.N + 1;
    const long long npe = (long long)nr * ns * nt;
    const long long fsE = a.nel * npe;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        const int gx = idx % X;
        const long long t = idx / X;
        const int gy = t % Y;
        const int gz = t / Y;
        int ex[2], ix[2], ey[2], iy[2], ez[2], iz[2];
        auto copies = [](int gi, int N, int ne, int* e, int* l) {
            if (gi > 0 && gi < ne * N && gi % N == 0) {
                e[0] = gi / N - 1; l[0] = N;
                e[1] = gi / N;     l[1] = 0;
                return 2;
            }
            e[0] = min(gi / N, ne - 1);
            l[0] = gi - e[0] * N;
            return 1;
        };
        const int cx = copies(gx, a.N, g.nex, ex, ix);
        const int cy = copies(gy, a.Ny, g.ney, ey, iy);
        const int cz = copies(gz, a.N, g.nez, ez, iz);
        for (int f = 0; f < nf; ++f) {
            double num = 0.0, den = 0.0;
            for (int c3 = 0; c3 < cz; ++c3)
                for (int c2 = 0; c2 < cy; ++c2)
                    for (int c1 = 0; c1 < cx; ++c1) {
                        const long long e = ((long long)ez[c3] * g.ney + ey[c2]) * g.nex + ex[c1];
                        const long long node = e * npe + ((long long)iz[c3] * ns + iy[c2]) * nr + ix[c1];
                        const double w = (Wx[ex[c1] * nr + ix[c1]] * Wy[ey[c2] * ns + iy[c2]]) *
                                         Wz[ez[c3] * nt + iz[c3]];
                        num += w * Ein[f * fsE + node];
                        den += w;
                    }
            const double v = num / den;
            for (int c3 = 0; c3 < cz; ++c3)
                for (int c2 = 0; c2 < cy; ++c2)
                    for (int c1 = 0; c1 < cx; ++c1) {
                        const long long e = ((long long)ez[c3] * g.ney + ey[c2]) * g.nex + ex[c1];
                        Eout[f * fsE + e * npe + ((long long)iz[c3] * ns + iy[c2]) * nr + ix[c1]] = v;
                    }
        }
    }
}

// ---------------------------------------------------------------------------
// generic batched banded column API
// ---------------------------------------------------------------------------
__device__ __forceinline__ long long bidx(int d, int k, int c, int M, int n_col) {
    return ((long long)d * M + k) * n_col + c;
}

__global__ void k_band_pack(const double* dense, double* band, int n_col, int M, int nb) {
    const int W = 2 * nb - 1;
    const long long n = (long long)n_col * M * W;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        const int c = idx % n_col;
        const long long t = idx / n_col;
        const int k = t % M;
        const int d = t / M;
        const int j = k + d - (nb - 1);
        band[idx] = (j >= 0 && j < M) ? dense[((long long)c * M + k) * M + j] : 0.0;
    }
}

__global__ void k_band_unpack(const double* band, double* dense, int n_col, int M, int nb) {
    const long long n = (long long)n_col * M * M;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        const int j = idx % M;
        const long long t = idx / M;
        const int k = t % M;
        const int c = t / M;
        const int d = j - k + nb - 1;
        dense[idx] = (d >= 0 && d < 2 * nb - 1) ? band[bidx(d, k, c, M, n_col)] : 0.0;
    }
}

__global__ void k_band_lu(double* B, int n_col, int M, int nb, double norm, int* bad) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_col) return;
    const int o = nb - 1;
    for (int k = 0; k < M; ++k) {
        double piv = B[bidx(o, k, c, M, n_col)];
        if (fabs(piv) < 1e-12 * norm) {
            atomicMin(bad, c);
            piv = 1.0;
        }
        const int E = min(k + nb, M);
        for (int r = k + 1; r < E; ++r) B[bidx(k - r + o, r, c, M, n_col)] /= piv;
        for (int r = k + 1; r < E; ++r) {
            const double l = B[bidx(k - r + o, r, c, M, n_col)];
            for (int cc = k + 1; cc < E; ++cc)
                B[bidx(cc - r + o, r, c, M, n_col)] -= l * B[bidx(cc - k + o, k, c, M, n_col)];
        }
    }
}

__global__ void k_band_solve(const double* B, double* rhs, int n_col, int M, int nb) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_col) return;
    const int o = nb - 1;
    double* y = rhs + (long long)c * M;
    for (int i = 1; i < M; ++i) {
        double s = 0.0;
        for (int j = max(0, i - nb + 1); j < i; ++j) s = fma(B[bidx(j - i + o, i, c, M, n_col)], y[j], s);
        y[i] -= s;
    }
    for (int i = M - 1; i >= 0; --i) {
        double s = 0.0;
        for (int j = i + 1; j < min(i + nb, M); ++j) s = fma(B[bidx(j - i + o, i, c, M, n_col)], y[j], s);
        y[i] = (y[i] - s) / B[bidx(o, i, c, M, n_col)];
    }
}

// Direct solve of the standard (5-variable) form, one thread per column
// (columnsolve.solve_direct, form="standard", columnsolve.py:196-204): the
// unknown i = lev*5 + field of a column is read straight from the lattice
// (coalesced across columns), one shared band LU (box columns are identical),
// forward / backward substitution in place in the output lattice.
__global__ void k_std_solve(const Geo g, int N, const double* __restrict__ B, int M, int nb,
                            const double* __restrict__ qe, double* __restrict__ q) {
    extern __shared__ double sB[];
    const int W = 2 * nb - 1;
    for (int i = threadIdx.x; i < W * M; i += blockDim.x) sB[i] = B[i];
    __syncthreads();
    const int NYo = g.slab ? 1 : N;
    const int cntx = (g.ex_e - g.ex_b) * N + (g.ex_e == g.nex ? 1 : 0);
    const int cnty = (g.ey_e - g.ey_b) * NYo + (g.ey_e == g.ney ? 1 : 0);
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cntx * cnty) return;
    const int gx = g.ex_b * N + c % cntx, gy = g.ey_b * NYo + c / cntx;
    const long long col = loff(g, gx, gy, 0);
    const long long ls = (long long)g.lY * g.px;
    auto at = [&](int i) { return (long long)(i % 5) * g.fs + (long long)(i / 5) * ls + col; };
    const int o = nb - 1;
    for (int i = 0; i < M; ++i) {
        double s = 0.0;
        for (int j = max(0, i - nb + 1); j < i; ++j) s = fma(sB[(j - i + o) * M + i], q[at(j)], s);
        q[at(i)] = qe[at(i)] - s;
    }
    for (int i = M - 1; i >= 0; --i) {
        double s = 0.0;
        for (int j = i + 1; j < min(i + nb, M); ++j) s = fma(sB[(j - i + o) * M + i], q[at(j)], s);
        q[at(i)] = (q[at(i)] - s) / sB[o * M + i];
    }
}

// Halo pack / unpack for the column-partitioned step (SURVEY 8(b)
// "halo_pack"): a region [xlo, xhi) x [ylo, yhi) (global lattice indices) of
// every level and nf fields <-> a contiguous (nf, Z, ny, nx) buffer, so one
// NCCL send/recv per neighbour moves it.
__global__ void k_halo(const Geo g, double* q, int nf, int xlo, int xhi, int ylo, int yhi,
                       double* buf, int unpack) {
    const int nx = xhi - xlo, ny = yhi - ylo;
    const long long n = (long long)nf * g.Z * ny * nx;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(i % nx);
        long long t = i / nx;
        const int y = (int)(t % ny);
        t /= ny;
        const int z = (int)(t % g.Z);
        const int f = (int)(t / g.Z);
        const long long o = f * g.fs + loff(g, xlo + x, ylo + y, z);
        if (unpack)
            q[o] = buf[i];
        else
            buf[i] = q[o];
    }
}

__global__ void k_absmax(const double* a, long long n, unsigned long long* out) {
    double m = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        m = fmax(m, fabs(a[i]));
    for (int s = 16; s > 0; s >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, s));
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

#include "explicit_v2.cuh"
#include "explicit_col.cuh"
#include "explicit_colc.cuh"
#include "explicit_c.cuh"
#include "solve_v2.cuh"
#include "imex3d.cuh"
#include "general.cuh"

// P' plane of a lattice state over the plan's whole window (stage 0 of the
// fused step: formed once per point here instead of for every staged,
// halo-overlapped point inside the explicit kernel)
struct BC16 {
    double v[16];
};

// grid (x blocks, rows y, levels z): the level constants once per thread
__global__ void __launch_bounds__(256) k_pp_plane(const Geo g, Lev lv, Phys ph, const double* __restrict__ q,
                                                  double* __restrict__ pp, const BC16 bcv) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= g.lX) return;
    const int k = blockIdx.z;
    const long long o = ((long long)k * g.lY + blockIdx.y) * g.px + x;
    const double r = q[o], th = q[o + 4 * g.fs];
    const double rho0 = __ldg(lv.rho0 + k), th0 = __ldg(lv.theta0 + k);
    const double delta = (r * th0 + th * (rho0 + r)) * __ldg(lv.irt0 + k);
    double v;
    if (HEVI_PP_SHORT && fabs(delta) <= 0x1p-10) {   // pprime (explicit_v2.cuh), short series
        double sum = bcv.v[5];
#pragma unroll
        for (int j = 4; j >= 0; --j) sum = fma(sum, delta, bcv.v[j]);
        v = fma(__ldg(lv.E0 + k), sum * delta, __ldg(lv.c0 + k));
    } else if (fabs(delta) <= 0.125) {   // the 15-term series branch
        double sum = bcv.v[14];
#pragma unroll
        for (int j = 13; j >= 0; --j) sum = fma(sum, delta, bcv.v[j]);
        v = fma(__ldg(lv.E0 + k), sum * delta, __ldg(lv.c0 + k));
    } else {
        v = pprime_pow(rho0 + r, th0 + th, __ldg(lv.P0f + k), ph.P0, ph.R, ph.gamma);
    }
    pp[o] = v;
}

}  // namespace

// ---------------------------------------------------------------------------
// plan
// ---------------------------------------------------------------------------
struct Factor {
    double lam = 0.0;
    int nb = 0;
    double* A = nullptr;       // M*M
    double* LU = nullptr;      // M*M
    double* LUb = nullptr;     // M*(2*M-1) upper bound
    double* lamtab = nullptr;  // 3*M
    double* vtab = nullptr;    // 12*M
    double* LU2 = nullptr;     // M*(4N+1)
    double* rU = nullptr;      // M
    double* rec = nullptr;     // M * RS: k_solve2's per-level records
    int* d_nb = nullptr;
    unsigned* d_bad = nullptr; // degenerate no-pivot diagonal seen
    int pivoted = 0;           // factor_with_fallback took the pivoted path
    double* LUP = nullptr;     // M*M pivoted dense LU
    int* piv = nullptr;        // M interchanges
    int* d_info = nullptr;
};

struct hevi_plan {
    Geo g;
    Lev lv;
    Phys ph;
    int N, Ny, ainv_identity;
    double* d_tab = nullptr;
    const double *cx, *cy, *cz, *Dx, *Dy, *Dz;
    unsigned* d_flags = nullptr;
    unsigned* h_flags = nullptr;
    std::map<long long, Factor> factors;
    double bc[16];
    double hDz[81];   // host copy of the vertical D matrix (the column kernels' parameter bank)
    int eqset = 0;   // 0: set2nc, 1: set2c
    int force_pivoted = 0;   // HEVI_OPT_FORCE_PIVOTED (tests of the fallback path)
    // the column solve of stage s wrote P' of its output into the P buffer's
    // field 1 + s of this workspace (the next explicit stage reads it)
    int pp_ok[2] = {0, 0};
    const double* pp_work = nullptr;
    unsigned long long* d_dbg = nullptr;
    bool use_v2 = true;
    bool use_tma = true;
    bool use_col = true;     // explicit_col kernels (3D, N = 4, set2nc)
    bool lt_ok = false;      // lt filled (Z <= EC_ZMAX)
    // fork/join of the domain-end kernel (k_ecol_edge) beside the main sweep:
    // it runs in the main kernel's last, partial wave (capturable in graphs)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    double* ppscratch = nullptr;   // hevi_rhs on the column sweep: P'(q) of the caller's state
    LvlTab lt;               // per-level constants of the explicit_col kernels
};

// general (curvilinear) mesh plan: per-column Schur factors
struct GFactor {
    double lam = 0.0;
    int nb = 0, pivoted = 0;
    double* A = nullptr;      // n_col x M x M probed matrices (kept for hevi_g_column_matrix)
    double* band = nullptr;   // n_col x M x (2nb-1) no-pivot banded LU (k_band_* layout)
    double* LUP = nullptr;    // pivoted dense LU per column (fallback)
    int* piv = nullptr;
};

struct hevi_gplan {
    GGeo g;
    GRef r;
    long long nn = 0;
    int n_groups = 0, n_proj = 0, n_col = 0, n_lev = 0;
    int *d_gptr = nullptr, *d_gidx = nullptr, *d_gslot = nullptr, *d_uid = nullptr, *d_rep = nullptr,
        *d_bslot = nullptr;
    double *d_w = nullptr, *d_wsum = nullptr;
    double* d_arr = nullptr;   // geometry and background arrays
    double* d_scr = nullptr;   // scratch: s0, s1, ua[3], up[3], sP, sO
    double *s0 = nullptr, *s1 = nullptr, *ua = nullptr, *up = nullptr, *sP = nullptr, *sO = nullptr;
    double* col = nullptr;     // n_col x n_lev column buffer
    unsigned* d_flags = nullptr;
    unsigned* h_flags = nullptr;
    unsigned long long* d_bits = nullptr;
    int* d_nb = nullptr;
    std::map<long long, GFactor> factors;
};

namespace {

long long lam_key(double lam) { return llround(lam * 1e12); }

// dynamic shared-memory opt-in of a kernel, per device (the attribute is
// per device: a process may drive several GPUs)
template <typename K>
int set_smem_attr(K kern, size_t smem, size_t (&done)[16]) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 16) return fail("device index out of range");
    if (done[dev] < smem) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        done[dev] = smem;
    }
    return HEVI_OK;
}

// ---- explicit-kernel dispatch -------------------------------------------
template <int NX, int NY>
struct TileCfg;
// 3D (Ny == N)
template <> struct TileCfg<1, 1> { static constexpr int TX = 8, TY = 8; };
template <> struct TileCfg<2, 2> { static constexpr int TX = 4, TY = 4; };
template <> struct TileCfg<3, 3> { static constexpr int TX = 3, TY = 3; };
template <> struct TileCfg<4, 4> { static constexpr int TX = 2, TY = 2; };
template <> struct TileCfg<5, 5> { static constexpr int TX = 2, TY = 1; };
template <> struct TileCfg<6, 6> { static constexpr int TX = 1, TY = 1; };
template <> struct TileCfg<7, 7> { static constexpr int TX = 1, TY = 1; };
template <> struct TileCfg<8, 8> { static constexpr int TX = 1, TY = 1; };
// slab (Ny == 1, one element across y); N == 1 slab coincides with the 3D N=1 case
template <> struct TileCfg<2, 1> { static constexpr int TX = 16, TY = 1; };
template <> struct TileCfg<3, 1> { static constexpr int TX = 12, TY = 1; };
template <> struct TileCfg<4, 1> { static constexpr int TX = 8, TY = 1; };
template <> struct TileCfg<5, 1> { static constexpr int TX = 6, TY = 1; };
template <> struct TileCfg<6, 1> { static constexpr int TX = 5, TY = 1; };
template <> struct TileCfg<7, 1> { static constexpr int TX = 4, TY = 1; };
template <> struct TileCfg<8, 1> { static constexpr int TX = 4, TY = 1; };

template <int NX, int NY, int MODE>
int launch_e(const hevi_plan* pl, EArgs a, cudaStream_t st) {
    constexpr int TX = TileCfg<NX, NY>::TX, TY = TileCfg<NX, NY>::TY;
    using T = ETile<NX, NY, NX, TX, TY>;
    auto kern = k_explicit<NX, NY, NX, TX, TY, MODE>;
    static size_t attr[16] = {0};
    int rc = set_smem_attr(kern, T::SMEM, attr);
    if (rc) return rc;
    const Geo& g = pl->g;
    dim3 grid((g.ex_e - g.ex_b + TX - 1) / TX, (g.ey_e - g.ey_b + TY - 1) / TY);
    kern<<<grid, T::BLK, T::SMEM, st>>>(a);
    CK(cudaGetLastError());
    return HEVI_OK;
}

template <int MODE>
int dispatch_e(const hevi_plan* pl, const EArgs& a, cudaStream_t st) {
    const int N = pl->N, Ny = pl->Ny;
    if (Ny == N) {
        switch (N) {
            case 1: return launch_e<DN(1), 1, MODE>(pl, a, st);
            case 2: return launch_e<DN(2), DN(2), MODE>(pl, a, st);
            case 3: return launch_e<DN(3), DN(3), MODE>(pl, a, st);
            case 4: return launch_e<DN(4), DN(4), MODE>(pl, a, st);
            case 5: return launch_e<DN(5), DN(5), MODE>(pl, a, st);
            case 6: return launch_e<DN(6), DN(6), MODE>(pl, a, st);
            case 7: return launch_e<DN(7), DN(7), MODE>(pl, a, st);
            case 8: return launch_e<DN(8), DN(8), MODE>(pl, a, st);
        }
    } else if (Ny == 1) {
        switch (N) {
            case 2: return launch_e<DN(2), 1, MODE>(pl, a, st);
            case 3: return launch_e<DN(3), 1, MODE>(pl, a, st);
            case 4: return launch_e<DN(4), 1, MODE>(pl, a, st);
            case 5: return launch_e<DN(5), 1, MODE>(pl, a, st);
            case 6: return launch_e<DN(6), 1, MODE>(pl, a, st);
            case 7: return launch_e<DN(7), 1, MODE>(pl, a, st);
            case 8: return launch_e<DN(8), 1, MODE>(pl, a, st);
        }
    }
    return fail("unsupported polynomial order (supported: N = 1..8; slab Ny = 1)");
}

// ---- v2 explicit dispatch (TMA ring-buffer kernel) ------------------------
template <int N, int NY>
struct Tile2 {
    static constexpr int TX = 0, TY = 0, MINB = 1;
};
template <> struct Tile2<1, 1> { static constexpr int TX = 16, TY = 16, MINB = 1; };
template <> struct Tile2<2, 2> { static constexpr int TX = 8, TY = 4, MINB = 1; };
template <> struct Tile2<3, 3> { static constexpr int TX = 4, TY = 2, MINB = 2; };
template <> struct Tile2<4, 4> { static constexpr int TX = HEVI_T44_TX, TY = HEVI_T44_TY, MINB = HEVI_T44_MINB; };
template <> struct Tile2<5, 5> { static constexpr int TX = 2, TY = 2, MINB = 1; };
template <> struct Tile2<6, 6> { static constexpr int TX = 2, TY = 1, MINB = 1; };
template <> struct Tile2<7, 7> { static constexpr int TX = 1, TY = 1, MINB = 1; };
template <> struct Tile2<2, 1> { static constexpr int TX = 32, TY = 1, MINB = 2; };
template <> struct Tile2<3, 1> { static constexpr int TX = 16, TY = 1, MINB = 2; };
template <> struct Tile2<4, 1> { static constexpr int TX = 8, TY = 1, MINB = 2; };
template <> struct Tile2<5, 1> { static constexpr int TX = 8, TY = 1, MINB = 1; };
template <> struct Tile2<6, 1> { static constexpr int TX = 6, TY = 1, MINB = 1; };
template <> struct Tile2<7, 1> { static constexpr int TX = 4, TY = 1, MINB = 1; };
template <> struct Tile2<8, 1> { static constexpr int TX = 4, TY = 1, MINB = 1; };

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                      const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                      const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                      CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled_t encode_fn() {
    static PFN_encodeTiled_t fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_encodeTiled_t)p;
    }
    return fn;
}

// 4D map (x, y, level, field) over a rank's lattice array, box = one layer tile
int make_tmap(CUtensorMap* m, const Geo& g, const double* base, int bx, int by, int bz, int nf = 5) {
    PFN_encodeTiled_t enc = encode_fn();
    if (!enc) return fail("cuTensorMapEncodeTiled unavailable");
    if (((uintptr_t)base & 15) || (g.px & 1)) return fail("lattice arrays must be 16-byte aligned with even pitch");
    cuuint64_t dims[4] = {(cuuint64_t)g.lX, (cuuint64_t)g.lY, (cuuint64_t)g.Z, (cuuint64_t)nf};
    cuuint64_t strides[3] = {(cuuint64_t)g.px * 8, (cuuint64_t)g.lY * g.px * 8, (cuuint64_t)g.fs * 8};
    cuuint32_t box[4] = {(cuuint32_t)bx, (cuuint32_t)by, (cuuint32_t)bz, (cuuint32_t)nf};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)base, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail("cuTensorMapEncodeTiled failed");
    return HEVI_OK;
}

template <int N, int NY, int MODE>
int launch_e2(const hevi_plan* pl, const EArgs& a, cudaStream_t st, bool& done) {
    constexpr int TX = Tile2<N, NY>::TX, TY = Tile2<N, NY>::TY;
    done = false;
    if constexpr (TX == 0) {
        return HEVI_OK;
    } else {
        using T = E2<N, NY, TX, TY>;
        const Geo& g = pl->g;
        const size_t smem = T::fixed_bytes(MODE) + sizeof(double) * T::NTAB * g.Z;
        if (smem > 225 * 1024) return HEVI_OK;   // v1 handles it
        auto kern = k_explicit2<N, NY, TX, TY, MODE, Tile2<N, NY>::MINB>;
        static size_t attr[16] = {0};
        int rc = set_smem_attr(kern, smem, attr);
        if (rc) return rc;
        CUtensorMap tm;
        rc = make_tmap(&tm, g, a.q, T::LXT, T::LY, 1);   // one level per TMA
        if (rc) return rc;
        EArgs a2 = a;
        a2.af_tma = 0;
        CUtensorMap tA = tm, tF = tm;
        if (T::AF_N > 0 && ((HEVI_X_AFTMA_MASK >> MODE) & 1) && (MODE == M_S2 || MODE == M_S3) && a.F &&
            (MODE == M_S3 || a.A) && (g.x0 % 2 == 0)) {
            if (MODE == M_S2) {
                rc = make_tmap(&tA, g, a.A, T::OX, T::OYM, N);
                if (rc) return rc;
            }
            rc = make_tmap(&tF, g, a.F, T::OX, T::OYM, N);
            if (rc) return rc;
            a2.af_tma = 1;
        }
        CUtensorMap tP = tm;
        if ((MODE == M_S1 || MODE == M_S2 || MODE == M_S3) && a.pp_in) {
            rc = make_tmap(&tP, g, a.pp_in, T::LXT, T::LY, 1, 1);   // one level of the P' plane
            if (rc) return rc;
        } else {
            a2.pp_in = nullptr;
        }
        dim3 grid((g.ex_e - g.ex_b + TX - 1) / TX, (g.ey_e - g.ey_b + TY - 1) / TY);
        kern<<<grid, T::BLK, smem, st>>>(a2, tm, tA, tF, tP);
        CK(cudaGetLastError());
        done = true;
        return HEVI_OK;
    }
}

template <int MODE>
int dispatch_e2(const hevi_plan* pl, const EArgs& a, cudaStream_t st, bool& done) {
    const int N = pl->N, Ny = pl->Ny;
    done = false;
    if (Ny == N) {
        switch (N) {
            case 1: return launch_e2<DN(1), 1, MODE>(pl, a, st, done);
            case 2: return launch_e2<DN(2), DN(2), MODE>(pl, a, st, done);
            case 3: return launch_e2<DN(3), DN(3), MODE>(pl, a, st, done);
            case 4: return launch_e2<DN(4), DN(4), MODE>(pl, a, st, done);
            case 5: return launch_e2<DN(5), DN(5), MODE>(pl, a, st, done);
            case 6: return launch_e2<DN(6), DN(6), MODE>(pl, a, st, done);
            case 7: return launch_e2<DN(7), DN(7), MODE>(pl, a, st, done);
        }
    } else if (Ny == 1) {
        switch (N) {
            case 2: return launch_e2<DN(2), 1, MODE>(pl, a, st, done);
            case 3: return launch_e2<DN(3), 1, MODE>(pl, a, st, done);
            case 4: return launch_e2<DN(4), 1, MODE>(pl, a, st, done);
            case 5: return launch_e2<DN(5), 1, MODE>(pl, a, st, done);
            case 6: return launch_e2<DN(6), 1, MODE>(pl, a, st, done);
            case 7: return launch_e2<DN(7), 1, MODE>(pl, a, st, done);
            case 8: return launch_e2<DN(8), 1, MODE>(pl, a, st, done);
        }
    }
    return HEVI_OK;
}

int run_e2(const hevi_plan* pl, int mode, const EArgs& a, cudaStream_t st, bool& done) {
    switch (mode) {
        case M_R: return dispatch_e2<M_R>(pl, a, st, done);
        case M_L: return dispatch_e2<M_L>(pl, a, st, done);
        case M_S1: return dispatch_e2<M_S1>(pl, a, st, done);
        case M_S2: return dispatch_e2<M_S2>(pl, a, st, done);
        case M_S3: return dispatch_e2<M_S3>(pl, a, st, done);
        case M_RK: return dispatch_e2<M_RK>(pl, a, st, done);
    }
    return fail("bad mode");
}

// ---- set2c explicit dispatch ---------------------------------------------
template <int N, int NY>
struct TileC {
    static constexpr int TX = 0, TY = 0;
};
template <> struct TileC<1, 1> { static constexpr int TX = 8, TY = 8; };
template <> struct TileC<2, 2> { static constexpr int TX = 4, TY = 4; };
template <> struct TileC<3, 3> { static constexpr int TX = 3, TY = 3; };
template <> struct TileC<4, 4> { static constexpr int TX = 2, TY = 2; };
template <> struct TileC<5, 5> { static constexpr int TX = 1, TY = 1; };
template <> struct TileC<6, 6> { static constexpr int TX = 1, TY = 1; };
template <> struct TileC<2, 1> { static constexpr int TX = 16, TY = 1; };
template <> struct TileC<3, 1> { static constexpr int TX = 12, TY = 1; };
template <> struct TileC<4, 1> { static constexpr int TX = 8, TY = 1; };
template <> struct TileC<5, 1> { static constexpr int TX = 6, TY = 1; };
template <> struct TileC<6, 1> { static constexpr int TX = 5, TY = 1; };
template <> struct TileC<7, 1> { static constexpr int TX = 4, TY = 1; };
template <> struct TileC<8, 1> { static constexpr int TX = 4, TY = 1; };

template <int N, int NY, int MODE>
int launch_c(const hevi_plan* pl, const EArgs& a, cudaStream_t st) {
    constexpr int TX = TileC<N, NY>::TX, TY = TileC<N, NY>::TY;
    if constexpr (TX == 0) {
        return fail("set2c: unsupported polynomial order for the device path");
    } else {
        using T = ECT<N, NY, TX, TY>;
        auto kern = k_explicit_c<N, NY, TX, TY, MODE>;
        static size_t attr[16] = {0};
        int rc = set_smem_attr(kern, T::SMEM, attr);
        if (rc) return rc;
        const Geo& g = pl->g;
        dim3 grid((g.ex_e - g.ex_b + TX - 1) / TX, (g.ey_e - g.ey_b + TY - 1) / TY);
        kern<<<grid, T::BLK, T::SMEM, st>>>(a);
        CK(cudaGetLastError());
        return HEVI_OK;
    }
}

template <int MODE>
int dispatch_c(const hevi_plan* pl, const EArgs& a, cudaStream_t st) {
    const int N = pl->N, Ny = pl->Ny;
    if (Ny == N) {
        switch (N) {
            case 1: return launch_c<DN(1), 1, MODE>(pl, a, st);
            case 2: return launch_c<DN(2), DN(2), MODE>(pl, a, st);
            case 3: return launch_c<DN(3), DN(3), MODE>(pl, a, st);
            case 4: return launch_c<DN(4), DN(4), MODE>(pl, a, st);
            case 5: return launch_c<DN(5), DN(5), MODE>(pl, a, st);
            case 6: return launch_c<DN(6), DN(6), MODE>(pl, a, st);
        }
    } else if (Ny == 1) {
        switch (N) {
            case 2: return launch_c<DN(2), 1, MODE>(pl, a, st);
            case 3: return launch_c<DN(3), 1, MODE>(pl, a, st);
            case 4: return launch_c<DN(4), 1, MODE>(pl, a, st);
            case 5: return launch_c<DN(5), 1, MODE>(pl, a, st);
            case 6: return launch_c<DN(6), 1, MODE>(pl, a, st);
            case 7: return launch_c<DN(7), 1, MODE>(pl, a, st);
            case 8: return launch_c<DN(8), 1, MODE>(pl, a, st);
        }
    }
    return fail("set2c: unsupported polynomial order for the device path");
}

#ifndef HEVI_SKIP_EDGE
#define HEVI_SKIP_EDGE 0   // timing experiments only: no domain-end kernel (wrong results)
#endif
// a launch that may overlap the stream's previous kernel once that kernel's
// CTAs have all executed griddepcontrol.launch_dependents
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), unsigned blocks, unsigned threads, cudaStream_t st,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---- explicit_col dispatch (3D box, N = 4, set2nc, stage kernels) --------
// cudaFuncSetAttribute once per (kernel, device)

bool col_applies(const hevi_plan* pl, int mode, const EArgs& a) {
    const Geo& g = pl->g;
    return pl->use_col && pl->use_tma && pl->lt_ok && pl->eqset == 0 && pl->N == 4 && pl->Ny == 4 &&
           !g.slab && (g.x0 % 2) == 0 && (g.px % 2) == 0 && a.pp_in != nullptr &&
           (mode == M_S1 || mode == M_S2 || mode == M_S3 || mode == M_R);
}

// 4D map over a 5-field lattice array whose box covers nf consecutive fields
// (the field coordinate of a copy selects the first one)
int make_tmap_fields(CUtensorMap* m, const Geo& g, const double* base, int bx, int by, int nf) {
    PFN_encodeTiled_t enc = encode_fn();
    if (!enc) return fail("cuTensorMapEncodeTiled unavailable");
    if (((uintptr_t)base & 15) || (g.px & 1)) return fail("lattice arrays must be 16-byte aligned with even pitch");
    cuuint64_t dims[4] = {(cuuint64_t)g.lX, (cuuint64_t)g.lY, (cuuint64_t)g.Z, 5};
    cuuint64_t strides[3] = {(cuuint64_t)g.px * 8, (cuuint64_t)g.lY * g.px * 8, (cuuint64_t)g.fs * 8};
    cuuint32_t box[4] = {(cuuint32_t)bx, (cuuint32_t)by, 1, (cuuint32_t)nf};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)base, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail("cuTensorMapEncodeTiled failed");
    return HEVI_OK;
}

// tile split of a rank window for overlapping the halo exchange with the
// sweep: a tile is on the ring when its staged box reaches a halo point a
// neighbour rank provides (low side: the first tile when ex_b > 0; high
// side: the last tile when ex_e < nex; the same in y); the rest is interior
void tile_split(const Geo& g, int TX, int TY, int tb[6]) {
    const int nbx = (g.ex_e - g.ex_b + TX - 1) / TX, nby = (g.ey_e - g.ey_b + TY - 1) / TY;
    const int bx0 = g.ex_b > 0 ? 1 : 0, by0 = g.ey_b > 0 ? 1 : 0;
    int bx1 = nbx - (g.ex_e < g.nex ? 1 : 0), by1 = nby - (g.ey_e < g.ney ? 1 : 0);
    if (bx1 < bx0) bx1 = bx0;
    if (by1 < by0) by1 = by0;
    tb[0] = nbx;
    tb[1] = nby;
    tb[2] = bx0;
    tb[3] = bx1;
    tb[4] = by0;
    tb[5] = by1;
}

// grid of the column-sweep launch for the tile subset of a.tmode (0 tiles: no launch)
dim3 tile_grid(EArgs& a, const Geo& g, int TX, int TY) {
    if (a.tmode == 0) return dim3((g.ex_e - g.ex_b + TX - 1) / TX, (g.ey_e - g.ey_b + TY - 1) / TY);
    tile_split(g, TX, TY, a.tb);
    const int ni = (a.tb[3] - a.tb[2]) * (a.tb[5] - a.tb[4]);
    if (a.tmode == 1) return ni ? dim3(a.tb[3] - a.tb[2], a.tb[5] - a.tb[4]) : dim3(0, 0);
    const int nr = a.tb[0] * a.tb[1] - ni;
    return dim3(nr, nr ? 1 : 0);
}

template <int N, int MODE>
int launch_col(const hevi_plan* pl, const EArgs& a0, cudaStream_t st) {
    using T = EC<N, MODE>;
    EArgs a = a0;
    const Geo& g = pl->g;
    static size_t attr[16] = {0};
    auto kern = k_ecol<N, MODE>;
    int rc = set_smem_attr(kern, T::SMEM, attr);
    if (rc) return rc;
    CUtensorMap tq, tp, tA, tF;
    if ((rc = make_tmap(&tq, g, a.q, T::LXT, T::LY, 1))) return rc;
    if ((rc = make_tmap(&tp, g, a.pp_in, T::LXT, T::LY, 1, 1))) return rc;
    tA = tq;
    tF = tq;
    if (MODE == M_S2 && (rc = make_tmap(&tA, g, a.A, T::OX, T::OY, 1))) return rc;
    if ((MODE == M_S2 || MODE == M_S3) && (rc = make_tmap(&tF, g, a.F, T::OX, T::OY, 1))) return rc;
    // TMA store destinations of stage 0's staged A and F (see EC::NOUT)
    CUtensorMap o0 = tq, o1 = tq, o2 = tq, o3 = tq;
    if (MODE == M_S1) {
        if ((rc = make_tmap_fields(&o0, g, a.A, T::OX, T::OY, 5))) return rc;
        if ((rc = make_tmap_fields(&o1, g, a.F, T::OX, T::OY, 5))) return rc;
    }
    // domain-end planes owned by this rank
    const int nxc = (g.ex_e == g.nex) ? (g.ey_e - g.ey_b) * N + (g.ey_e == g.ney ? 1 : 0) : 0;
    const int nyr = (g.ey_e == g.ney) ? (g.ex_e - g.ex_b) * N : 0;
    const long long npt = (long long)(nxc + nyr) * g.Z;
    // a partial tile at a domain end stores whole staging boxes, which cover
    // the domain-end plane: the edge kernel must then run after the sweep
    const bool partial_end = ((g.ex_e == g.nex) && (g.ex_e - g.ex_b) % T::TX != 0) ||
                             ((g.ey_e == g.ney) && (g.ey_e - g.ey_b) % T::TY != 0);
    const dim3 grid = tile_grid(a, g, T::TX, T::TY);
    const bool edge = !HEVI_SKIP_EDGE && npt > 0 && a.tmode != 1;   // the interior subset has no domain-end plane
    // the domain-end kernel as a programmatic dependent launch of the sweep
    // (starts once every sweep tile is resident; completes after the sweep)
    const bool pdl = HEVI_EDGE_PDL_NC && edge && grid.x && grid.y && !(T::NOUT && partial_end);
    const bool fork = !pdl && edge && pl->side != nullptr && !(T::NOUT && partial_end);
    if (fork) CK(cudaEventRecord(pl->ev_fork, st));
    if (grid.x && grid.y) {
        kern<<<grid, T::BLK, T::SMEM, st>>>(a, pl->lt, tq, tp, tA, tF, o0, o1, o2, o3);
        CK(cudaGetLastError());
    }
    if (pdl) {
        CK(launch_pdl(k_ecol_edge<N, MODE>, (unsigned)((npt + 127) / 128), 128, st, a, pl->lt, nxc, nyr,
                      g.ex_b * N, g.ey_b * N));
    } else if (edge) {
        // launched after the sweep: its blocks are dispatched as the sweep's last CTAs retire
        cudaStream_t es = fork ? pl->side : st;
        if (fork) CK(cudaStreamWaitEvent(es, pl->ev_fork, 0));
        k_ecol_edge<N, MODE><<<(unsigned)((npt + 127) / 128), 128, 0, es>>>(a, pl->lt, nxc, nyr, g.ex_b * N,
                                                                          g.ey_b * N);
        CK(cudaGetLastError());
        if (fork) {
            CK(cudaEventRecord(pl->ev_join, es));
            CK(cudaStreamWaitEvent(st, pl->ev_join, 0));
        }
    }
    return HEVI_OK;
}

// set2c column sweep (explicit_colc.cuh): no P' plane (formed per level in the kernel)
template <int N, int MODE>
int launch_colc(const hevi_plan* pl, const EArgs& a0, cudaStream_t st) {
    using T = ECC<N, MODE>;
    const Geo& g = pl->g;
    EArgs a = a0;
    a.pp_out = nullptr;
    static size_t attr[16] = {0};
    auto kern = k_ecolc<N, MODE>;
    int rc = set_smem_attr(kern, T::SMEM, attr);
    if (rc) return rc;
    CUtensorMap tq, tA, tF;
    if ((rc = make_tmap(&tq, g, a.q, T::LXT, T::LY, 1))) return rc;
    tA = tq;
    tF = tq;
    if (MODE == M_S2 && (rc = make_tmap(&tA, g, a.A, T::OX, T::OY, 1))) return rc;
    if ((MODE == M_S2 || MODE == M_S3) && (rc = make_tmap(&tF, g, a.F, T::OX, T::OY, 1))) return rc;
    const int nxc = (g.ex_e == g.nex) ? (g.ey_e - g.ey_b) * N + (g.ey_e == g.ney ? 1 : 0) : 0;
    const int nyr = (g.ey_e == g.ney) ? (g.ex_e - g.ex_b) * N : 0;
    const long long npt = (long long)(nxc + nyr) * g.Z;
    const dim3 grid = tile_grid(a, g, T::TX, T::TY);
    const bool edge = npt > 0 && a.tmode != 1;
    const bool pdl = HEVI_EDGE_PDL_C && edge && grid.x && grid.y;
    const bool fork = !pdl && edge && pl->side != nullptr;
    if (fork) CK(cudaEventRecord(pl->ev_fork, st));
    if (grid.x && grid.y) {
        kern<<<grid, T::BLK, T::SMEM, st>>>(a, pl->lt, tq, tA, tF);
        CK(cudaGetLastError());
    }
    if (pdl) {
        CK(launch_pdl(k_ecolc_edge<N, MODE>, (unsigned)((npt + 127) / 128), 128, st, a, pl->lt, nxc, nyr,
                      g.ex_b * N, g.ey_b * N));
    } else if (edge) {
        cudaStream_t es = fork ? pl->side : st;
        if (fork) CK(cudaStreamWaitEvent(es, pl->ev_fork, 0));
        k_ecolc_edge<N, MODE><<<(unsigned)((npt + 127) / 128), 128, 0, es>>>(a, pl->lt, nxc, nyr, g.ex_b * N,
                                                                           g.ey_b * N);
        CK(cudaGetLastError());
        if (fork) {
            CK(cudaEventRecord(pl->ev_join, es));
            CK(cudaStreamWaitEvent(st, pl->ev_join, 0));
        }
    }
    return HEVI_OK;
}

bool colc_applies(const hevi_plan* pl, int mode) {
    const Geo& g = pl->g;
    return pl->use_col && pl->use_tma && pl->lt_ok && pl->eqset == 1 && pl->N == 4 && pl->Ny == 4 &&
           !g.slab && (g.x0 % 2) == 0 && (g.px % 2) == 0 &&
           (mode == M_S1 || mode == M_S2 || mode == M_S3 || mode == M_R);
}

int run_colc(const hevi_plan* pl, int mode, const EArgs& a, cudaStream_t st) {
    switch (mode) {
        case M_R: return launch_colc<4, M_R>(pl, a, st);
        case M_S1: return launch_colc<4, M_S1>(pl, a, st);
        case M_S2: return launch_colc<4, M_S2>(pl, a, st);
        case M_S3: return launch_colc<4, M_S3>(pl, a, st);
    }
    return fail("bad mode");
}

int run_col(const hevi_plan* pl, int mode, const EArgs& a, cudaStream_t st) {
    switch (mode) {
        case M_R: return launch_col<4, M_R>(pl, a, st);
        case M_S1: return launch_col<4, M_S1>(pl, a, st);
        case M_S2: return launch_col<4, M_S2>(pl, a, st);
        case M_S3: return launch_col<4, M_S3>(pl, a, st);
    }
    return fail("bad mode");
}

int run_e(const hevi_plan* pl, int mode, const EArgs& a, cudaStream_t st) {
    if (a.tmode && !colc_applies(pl, mode) && !(pl->eqset == 0 && col_applies(pl, mode, a))) {
        // no tile split on this path: the boundary call does the whole stage
        if (a.tmode == 1) return HEVI_OK;
        EArgs b = a;
        b.tmode = 0;
        return run_e(pl, mode, b, st);
    }
    if (colc_applies(pl, mode)) return run_colc(pl, mode, a, st);
    if (pl->eqset == 1) {
        switch (mode) {
            case M_R: return dispatch_c<M_R>(pl, a, st);
            case M_L: return dispatch_c<M_L>(pl, a, st);
            case M_S1: return dispatch_c<M_S1>(pl, a, st);
            case M_S2: return dispatch_c<M_S2>(pl, a, st);
            case M_S3: return dispatch_c<M_S3>(pl, a, st);
            case M_RK: return dispatch_c<M_RK>(pl, a, st);
        }
        return fail("bad mode");
    }
    if (col_applies(pl, mode, a)) return run_col(pl, mode, a, st);
    if (pl->use_v2 && (pl->g.px % 2) == 0) {
        bool done = false;
        int rc = run_e2(pl, mode, a, st, done);
        if (rc || done) return rc;
    }
    switch (mode) {
        case M_R: return dispatch_e<M_R>(pl, a, st);
        case M_L: return dispatch_e<M_L>(pl, a, st);
        case M_S1: return dispatch_e<M_S1>(pl, a, st);
        case M_S2: return dispatch_e<M_S2>(pl, a, st);
        case M_S3: return dispatch_e<M_S3>(pl, a, st);
        case M_RK: return dispatch_e<M_RK>(pl, a, st);
    }
    return fail("bad mode");
}

EArgs base_eargs(const hevi_plan* pl) {
    EArgs a;
    memset(&a, 0, sizeof(a));
    a.g = pl->g;
    a.lv = pl->lv;
    a.ph = pl->ph;
    a.cx = pl->cx;
    a.cy = pl->cy;
    a.cz = pl->cz;
    a.Dx = pl->Dx;
    a.Dy = pl->Dy;
    a.Dz = pl->Dz;
    a.flags = pl->d_flags;
    memcpy(a.bc, pl->bc, sizeof(a.bc));
    a.use_tma = pl->use_tma ? 1 : 0;
    a.dbg = pl->d_dbg;
    return a;
}

// ---- column-kernel dispatch ---------------------------------------------
template <int NZ>
int launch_s(const hevi_plan* pl, SArgs a, cudaStream_t st) {
    const Geo& g = pl->g;
    const int M = g.Z;
    const int W = 2 * a.nb - 1;
    const size_t fixed = sizeof(double) * ((size_t)10 * M + (size_t)M * W + (NZ + 1) * (NZ + 1));
    int T = 128;
    while (T > 32 && fixed + sizeof(double) * 2 * (size_t)M * T > 200 * 1024) T /= 2;
    const size_t smem = fixed + sizeof(double) * 2 * (size_t)M * T;
    if (smem > 227 * 1024) return fail("column too tall for the shared-memory column kernel");
    static size_t attr[16] = {0};
    int rc = set_smem_attr(k_solve<NZ>, 227 * 1024, attr);
    if (rc) return rc;
    const int NYo = g.slab ? 1 : pl->N;
    const long long cntx = (long long)(g.ex_e - g.ex_b) * pl->N + (g.ex_e == g.nex ? 1 : 0);
    const long long cnty = (long long)(g.ey_e - g.ey_b) * NYo + (g.ey_e == g.ney ? 1 : 0);
    const long long ncol = cntx * cnty;
    const int blocks = (int)((ncol + T - 1) / T);
    k_solve<NZ><<<blocks, T, smem, st>>>(a);
    CK(cudaGetLastError());
    return HEVI_OK;
}

const Factor* find_factor(const hevi_plan* pl, double lam) {
    auto it = pl->factors.find(lam_key(lam));
    return it == pl->factors.end() ? nullptr : &it->second;
}

template <int N>
int launch_s2(const hevi_plan* pl, const Factor* f, const SArgs& a1, cudaStream_t st) {
    const Geo& g = pl->g;
    const int M = g.Z;
    S2Args a;
    memset(&a, 0, sizeof(a));
    a.g = g;
    a.ph = pl->ph;
    a.tab = f->vtab;
    a.LU2 = f->LU2;
    a.rU = f->rU;
    a.Dz = pl->Dz;
    memcpy(a.Dzc, pl->hDz, sizeof(a.Dzc));
    a.ainv_identity = pl->ainv_identity;
    a.lam = f->lam;
    a.P = a1.P;
    a.out = a1.out;
    a.src_uv = a1.src_uv;
    a.pp_out = a1.pp_out;
    a.lv = pl->lv;
    a.rec = f->rec;
    memcpy(a.bc, pl->bc, sizeof(a.bc));
    const int T = 128;
    if (f->pivoted) {   // columnsolve.factor_with_fallback: pivoted dense factor
        a.LU2 = f->LUP;
        const size_t smp = sizeof(double) * ((size_t)V_NT * M + (size_t)M * M + (N + 1) * (N + 1) +
                                             6 * (size_t)M + (size_t)M * T) + sizeof(int) * M;
        if (smp > 225 * 1024) return fail("column too tall for the pivoted column kernel");
        auto kern = pl->eqset == 1 ? k_solve_piv<N, true> : k_solve_piv<N, false>;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smp));
        const int NYp = g.slab ? 1 : pl->N;
        const long long nc = ((long long)(g.ex_e - g.ex_b) * pl->N + (g.ex_e == g.nex ? 1 : 0)) *
                             ((long long)(g.ey_e - g.ey_b) * NYp + (g.ey_e == g.ney ? 1 : 0));
        kern<<<(int)((nc + T - 1) / T), T, smp, st>>>(a, f->piv);
        CK(cudaGetLastError());
        return HEVI_OK;
    }
    const size_t smem = s2_smem_bytes<N>(M, T);
    if (smem > 225 * 1024) return fail("column too tall for the v2 column kernel");
    static size_t attr[16] = {0};
    int rc = set_smem_attr(k_solve2<N, false>, smem, attr);
    if (rc) return rc;
    const int NYo = g.slab ? 1 : pl->N;
    const long long cntx = (long long)(g.ex_e - g.ex_b) * pl->N + (g.ex_e == g.nex ? 1 : 0);
    const long long cnty = (long long)(g.ey_e - g.ey_b) * NYo + (g.ey_e == g.ney ? 1 : 0);
    const int nblk = (int)((cntx * cnty + T - 1) / T);
    if (pl->eqset == 1) {
        static size_t attrc[16] = {0};
        if ((rc = set_smem_attr(k_solve2<N, true>, smem, attrc))) return rc;
    }
    auto kern = pl->eqset == 1 ? k_solve2<N, true> : k_solve2<N, false>;
    // persistent grid: every resident CTA slot once (the records load once per CTA)
    int per_sm = 0, dev = 0, nsm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, smem));
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const int blocks = std::max(1, std::min(nblk, per_sm * nsm));
    kern<<<blocks, T, smem, st>>>(a);
    CK(cudaGetLastError());
    return HEVI_OK;
}

int run_s2(const hevi_plan* pl, const Factor* f, const SArgs& a, cudaStream_t st, bool& done) {
    done = false;
    if (!pl->use_v2 || (f->nb > 2 * pl->N + 1 && !f->pivoted)) return HEVI_OK;
    const size_t need = sizeof(double) * ((size_t)pl->g.Z * (4 * pl->N + 2 + (V_NT + 1) / 2 * 2 + 6 + 128) +
                                          (size_t)(pl->N + 1) * (pl->N + 1));   // s2_smem_bytes
    if (need > 220 * 1024) return HEVI_OK;
    int rc = HEVI_OK;
    switch (pl->N) {
        case 1: rc = launch_s2<DN(1)>(pl, f, a, st); break;
        case 2: rc = launch_s2<DN(2)>(pl, f, a, st); break;
        case 3: rc = launch_s2<DN(3)>(pl, f, a, st); break;
        case 4: rc = launch_s2<DN(4)>(pl, f, a, st); break;
        case 5: rc = launch_s2<DN(5)>(pl, f, a, st); break;
        case 6: rc = launch_s2<DN(6)>(pl, f, a, st); break;
        case 7: rc = launch_s2<DN(7)>(pl, f, a, st); break;
        case 8: rc = launch_s2<DN(8)>(pl, f, a, st); break;
        default: return HEVI_OK;
    }
    done = (rc == HEVI_OK);
    return rc;
}

int run_s(const hevi_plan* pl, const SArgs& a, cudaStream_t st, bool* v2 = nullptr) {
    if (v2) *v2 = false;
    {
        if (pl->eqset == 1) {
            const Factor* f = find_factor(pl, a.lam);
            bool done = false;
            int rc = f ? run_s2(pl, f, a, st, done) : fail("lam not factored");
            if (rc) return rc;
            if (!done) return fail("set2c: column too tall for the device column kernel");
            return HEVI_OK;
        }
        const Factor* f = find_factor(pl, a.lam);
        bool done = false;
        if (f) {
            int rc = run_s2(pl, f, a, st, done);
            if (v2) *v2 = done && rc == HEVI_OK;
            if (rc || done) return rc;
            if (f->pivoted) return fail("pivoted column factor needs the v2 column kernel");
        }
    }
    switch (pl->N) {
        case 1: return launch_s<DN(1)>(pl, a, st);
        case 2: return launch_s<DN(2)>(pl, a, st);
        case 3: return launch_s<DN(3)>(pl, a, st);
        case 4: return launch_s<DN(4)>(pl, a, st);
        case 5: return launch_s<DN(5)>(pl, a, st);
        case 6: return launch_s<DN(6)>(pl, a, st);
        case 7: return launch_s<DN(7)>(pl, a, st);
        case 8: return launch_s<DN(8)>(pl, a, st);
    }
    return fail("unsupported polynomial order");
}


SArgs base_sargs(const hevi_plan* pl, const Factor* f) {
    SArgs a;
    memset(&a, 0, sizeof(a));
    a.g = pl->g;
    a.lv = pl->lv;
    a.ph = pl->ph;
    a.cz = pl->cz;
    a.Dz = pl->Dz;
    a.LUb = f->LUb;
    a.lamtab = f->lamtab;
    a.nb = f->nb;
    a.ainv_identity = pl->ainv_identity;
    a.lam = f->lam;
    return a;
}

int blocks_for(long long n, int T = 256) {
    long long b = (n + T - 1) / T;
    if (b > 148LL * 32) b = 148LL * 32;
    if (b < 1) b = 1;
    return (int)b;
}

#include "general_host.cuh"

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* hevi_last_error(void) { return g_err.c_str(); }

#if defined(HEVI_PHASE_TIMING) || defined(HEVI_EDGE_TIMING)
// debug builds only: per-phase clock64 sums of the explicit kernel, reset after read
int hevi_debug_phase(hevi_plan* pl, unsigned long long* out8) {
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(out8, pl->d_dbg, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    CK(cudaMemset(pl->d_dbg, 0, 8 * sizeof(unsigned long long)));
    return HEVI_OK;
}
#endif

int hevi_plan_create(hevi_plan** out, const hevi_grid_desc* gd, const hevi_ref_desc* rd) {
    if (!out || !gd || !rd) return fail("null argument");
    *out = nullptr;
    if (gd->N < 1 || gd->N > 8) return fail("polynomial order must be in 1..8");
    if (!(gd->Ny == gd->N || gd->Ny == 1)) return fail("Ny must equal N (3D) or 1 (slab)");
    if (gd->slab && (gd->Ny != 1 || gd->ney != 1)) return fail("slab requires Ny = 1, ney = 1");
    if (gd->nex < 1 || gd->ney < 1 || gd->nez < 1) return fail("element counts must be >= 1");
    hevi_plan* pl = new hevi_plan();
    Geo& g = pl->g;
    g.nex = gd->nex;
    g.ney = gd->ney;
    g.nez = gd->nez;
    g.X = gd->nex * gd->N + 1;
    g.Y = gd->ney * gd->Ny + 1;
    g.Z = gd->nez * gd->N + 1;
    g.x0 = gd->x0;
    g.y0 = gd->y0;
    g.lX = gd->lX;
    g.lY = gd->lY;
    g.px = gd->px;
    g.fs = (long long)g.Z * g.lY * g.px;
    g.ex_b = gd->ex_b;
    g.ex_e = gd->ex_e;
    g.ey_b = gd->ey_b;
    g.ey_e = gd->ey_e;
    g.slab = gd->slab;
    if (g.px < g.lX || g.ex_b < 0 || g.ex_e > g.nex || g.ex_b >= g.ex_e || g.ey_b < 0 ||
        g.ey_e > g.ney || g.ey_b >= g.ey_e) {
        delete pl;
        return fail("inconsistent window / ownership");
    }
    pl->N = gd->N;
    pl->Ny = gd->Ny;
    pl->ph = {rd->g, rd->R, rd->P0, rd->gamma};
    const int Z = g.Z, X = g.X, Y = g.Y;
    const int nd = (gd->N + 1) * (gd->N + 1), ndy = (gd->Ny + 1) * (gd->Ny + 1);
    std::vector<double> h;
    h.reserve(9 * Z + X + Y + Z + 2 * nd + ndy);
    const double* lv[9] = {rd->rho0, rd->theta0, rd->P0f, rd->drho0, rd->dtheta0,
                           rd->G0,   rd->H0,     rd->F0z, rd->rho0G0};
    for (int t = 0; t < 9; ++t) h.insert(h.end(), lv[t], lv[t] + Z);
    h.insert(h.end(), rd->cx, rd->cx + X);
    h.insert(h.end(), rd->cy, rd->cy + Y);
    h.insert(h.end(), rd->cz, rd->cz + Z);
    h.insert(h.end(), rd->Dx, rd->Dx + nd);
    h.insert(h.end(), rd->Dy, rd->Dy + ndy);
    h.insert(h.end(), rd->Dz, rd->Dz + nd);
    memcpy(pl->hDz, rd->Dz, sizeof(double) * nd);
    // EOS reference point per level: Pb = EOS(rho0, theta0), c0 = Pb - P0f, 1/(rho0 theta0)
    h.insert(h.end(), rd->Pb, rd->Pb + Z);
    for (int k = 0; k < Z; ++k) h.push_back(rd->Pb[k] - rd->P0f[k]);
    for (int k = 0; k < Z; ++k) h.push_back(1.0 / (rd->rho0[k] * rd->theta0[k]));
    // set2c: Theta0, 1/Theta0, F0 (euler.py:103-113)
    h.insert(h.end(), rd->Theta0, rd->Theta0 + Z);
    for (int k = 0; k < Z; ++k) h.push_back(1.0 / rd->Theta0[k]);
    h.insert(h.end(), rd->F0c, rd->F0c + Z);
    pl->eqset = rd->eqset;
    if (rd->eqset != 0 && rd->eqset != 1) {
        delete pl;
        return fail("eqset must be 0 (set2nc) or 1 (set2c)");
    }
    pl->ainv_identity = 1;
    for (int k = 0; k < Z; ++k)
        if (rd->dtheta0[k] != 0.0) pl->ainv_identity = 0;
    cudaError_t e = cudaMalloc(&pl->d_tab, h.size() * sizeof(double));
    if (e == cudaSuccess) e = cudaMemcpy(pl->d_tab, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&pl->d_flags, 16 * sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMemset(pl->d_flags, 0, 16 * sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMallocHost(&pl->h_flags, 16 * sizeof(unsigned));
    if (e == cudaSuccess && getenv("HEVI_NO_FORK") == nullptr) {
        e = cudaStreamCreateWithFlags(&pl->side, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&pl->ev_fork, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&pl->ev_join, cudaEventDisableTiming);
    }
#if defined(HEVI_PHASE_TIMING) || defined(HEVI_EDGE_TIMING)
    if (e == cudaSuccess) e = cudaMalloc(&pl->d_dbg, 8 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemset(pl->d_dbg, 0, 8 * sizeof(unsigned long long));
#endif
    if (e != cudaSuccess) {
        hevi_plan_destroy(pl);
        return fail("plan allocation", e);
    }
    const double* d = pl->d_tab;
    pl->cx = d + 9 * Z;
    pl->cy = pl->cx + X;
    pl->cz = pl->cy + Y;
    pl->Dx = pl->cz + Z;
    pl->Dy = pl->Dx + nd;
    pl->Dz = pl->Dy + ndy;
    const double* eos = pl->Dz + nd;
    pl->lv = {d,         d + Z,     d + 2 * Z, d + 3 * Z, d + 4 * Z, d + 5 * Z,
              d + 6 * Z, d + 7 * Z, d + 8 * Z, eos,       eos + Z,   eos + 2 * Z,
              eos + 3 * Z, eos + 4 * Z, eos + 5 * Z};
    // binomial coefficients C(gamma, k) of the P' series
    {
        double cb = 1.0;
        for (int k = 1; k <= 15; ++k) {
            cb = cb * (rd->gamma - (k - 1)) / k;
            pl->bc[k - 1] = cb;
        }
        pl->bc[15] = 0.0;
    }
    pl->use_v2 = getenv("HEVI_KERNELS") == nullptr || strcmp(getenv("HEVI_KERNELS"), "v1") != 0;
    pl->use_tma = getenv("HEVI_NO_TMA") == nullptr;
    pl->use_col = pl->use_v2 && (getenv("HEVI_KERNELS") == nullptr || strcmp(getenv("HEVI_KERNELS"), "v2") != 0);
    if (Z <= EC_ZMAX && gd->N <= EC_NMAX && gd->Ny == gd->N) {
        LvlTab& t = pl->lt;
        memset(&t, 0, sizeof(t));
        for (int k = 0; k < Z; ++k) {
            t.v[C_RHO0][k] = rd->rho0[k];
            t.v[C_TH0][k] = rd->theta0[k];
            t.v[C_DRHO0][k] = rd->drho0[k];
            t.v[C_DTH0][k] = rd->dtheta0[k];
            t.v[C_CZ][k] = rd->cz[k];
            t.v[C_IRHO0][k] = 1.0 / rd->rho0[k];
            t.v[C_G0][k] = rd->G0[k];
            t.v[C_H0][k] = rd->H0[k];
            t.v[C_PB][k] = rd->Pb[k];
            t.v[C_C0][k] = rd->Pb[k] - rd->P0f[k];
            t.v[C_IRT0][k] = 1.0 / (rd->rho0[k] * rd->theta0[k]);
            t.v[C_P0F][k] = rd->P0f[k];
            t.v[C_TH0C][k] = rd->Theta0[k];
            t.v[C_ITH0][k] = 1.0 / rd->Theta0[k];
            t.v[C_F0C][k] = rd->F0c[k];
        }
        memcpy(t.dx, rd->Dx, sizeof(double) * nd);
        memcpy(t.dy, rd->Dy, sizeof(double) * ndy);
        memcpy(t.dz, rd->Dz, sizeof(double) * nd);
        const int N = gd->N;
        for (int k = 0; k < Z; ++k) {
            const int row = (k == Z - 1) ? N : k % N;
            const int base = k - row;
            for (int m = 0; m <= N; ++m) {
                t.dzs[k][m] = rd->cz[k] * rd->Dz[row * (N + 1) + m];
                t.pg[k][m] = t.dzs[k][m] * rd->G0[base + m];
                t.ph[k][m] = t.dzs[k][m] * rd->H0[base + m];
                if (k + m < Z) {
                    t.cg[k][m] = rd->Dz[N * (N + 1) + m] * rd->G0[k + m];
                    t.ch[k][m] = rd->Dz[N * (N + 1) + m] * rd->H0[k + m];
                }
            }
            t.czf[k] = (row == 0 && k > 0) ? rd->cz[k] : 0.0;
        }
        pl->lt_ok = true;
    }
    *out = pl;
    return HEVI_OK;
}

int hevi_plan_destroy(hevi_plan* pl) {
    if (!pl) return HEVI_OK;
    for (auto& kv : pl->factors) {
        cudaFree(kv.second.A);
        cudaFree(kv.second.LU);
        cudaFree(kv.second.LUb);
        cudaFree(kv.second.lamtab);
        cudaFree(kv.second.vtab);
        cudaFree(kv.second.LU2);
        cudaFree(kv.second.rU);
        cudaFree(kv.second.rec);
        cudaFree(kv.second.d_nb);
        cudaFree(kv.second.d_bad);
        cudaFree(kv.second.LUP);
        cudaFree(kv.second.piv);
        cudaFree(kv.second.d_info);
    }
    if (pl->ppscratch) cudaFree(pl->ppscratch);
    if (pl->side) cudaStreamDestroy(pl->side);
    if (pl->ev_fork) cudaEventDestroy(pl->ev_fork);
    if (pl->ev_join) cudaEventDestroy(pl->ev_join);
    cudaFree(pl->d_tab);
    cudaFree(pl->d_flags);
    if (pl->h_flags) cudaFreeHost(pl->h_flags);
    delete pl;
    return HEVI_OK;
}

long long hevi_state_size(const hevi_plan* pl) { return pl ? 5 * pl->g.fs : 0; }

int hevi_factor(hevi_plan* pl, double lam, int* nb_out, void* stream) {
    if (!pl) return fail("null plan");
    if (!(lam > 0.0)) return fail("implicit solve requires positive lam");
    cudaStream_t st = (cudaStream_t)stream;
    auto it = pl->factors.find(lam_key(lam));
    if (it == pl->factors.end()) {
        Factor f;
        f.lam = lam;
        const int M = pl->g.Z;
        if (pl->N > 16) return fail("order too high for probing");
        CK(cudaMalloc(&f.A, sizeof(double) * M * M));
        CK(cudaMalloc(&f.LU, sizeof(double) * M * M));
        CK(cudaMalloc(&f.LUb, sizeof(double) * M * (2 * M - 1)));
        CK(cudaMalloc(&f.lamtab, sizeof(double) * 3 * M));
        CK(cudaMalloc(&f.vtab, sizeof(double) * V_NT * M));
        CK(cudaMalloc(&f.LU2, sizeof(double) * M * (4 * pl->N + 1)));
        CK(cudaMalloc(&f.rU, sizeof(double) * M));
        CK(cudaMalloc(&f.d_nb, sizeof(int)));
        CK(cudaMalloc(&f.d_bad, sizeof(unsigned)));
        CK(cudaMemsetAsync(f.d_bad, 0, sizeof(unsigned), st));
        CK(cudaMemsetAsync(f.A, 0, sizeof(double) * M * M, st));
        FArgs a;
        a.lv = pl->lv;
        a.g = pl->ph.g;
        a.lam = lam;
        a.cz = pl->cz;
        a.Dz = pl->Dz;
        a.N = pl->N;
        a.nez = pl->g.nez;
        a.M = M;
        a.ainv_identity = pl->ainv_identity;
        a.eqset = pl->eqset;
        a.lamtab = f.lamtab;
        a.vtab = f.vtab;
        a.A = f.A;
        a.flags = pl->d_flags;
        k_lamtab<<<(M + 127) / 128, 128, 0, st>>>(a);
        CK(cudaGetLastError());
        k_probe<<<(M + 63) / 64, 64, 0, st>>>(a);
        CK(cudaGetLastError());
        k_lu_dense<<<1, 256, 0, st>>>(f.A, f.LU, f.LUb, M, f.d_nb, f.d_bad, pl->N, f.LU2, f.rU);
        CK(cudaGetLastError());
        {
            const int RS = 4 * pl->N + 2 + (V_NT + 1) / 2 * 2 + 6;
            CK(cudaMalloc(&f.rec, sizeof(double) * M * RS));
            k_s2rec<<<(M * RS + 255) / 256, 256, 0, st>>>(f.LU2, f.rU, f.vtab, pl->lv, M, pl->N, f.rec);
            CK(cudaGetLastError());
        }
        unsigned bad = 0;
        CK(cudaMemcpyAsync(&f.nb, f.d_nb, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&bad, f.d_bad, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (bad || pl->force_pivoted) {
            // columnsolve.factor_with_fallback (:141-153): keep a pivoted dense LU
            CK(cudaMalloc(&f.LUP, sizeof(double) * M * M));
            CK(cudaMalloc(&f.piv, sizeof(int) * M));
            CK(cudaMalloc(&f.d_info, sizeof(int)));
            k_lu_pivot<<<1, 256, 0, st>>>(f.A, f.LUP, f.piv, M, f.d_info);
            CK(cudaGetLastError());
            CK(cudaStreamSynchronize(st));
            f.pivoted = 1;
        }
        it = pl->factors.emplace(lam_key(lam), f).first;
    }
    if (nb_out) *nb_out = it->second.nb;
    return HEVI_OK;
}

int hevi_column_matrix(hevi_plan* pl, double lam, double* A_host, double* LU_host, void* stream) {
    const Factor* f = pl ? find_factor(pl, lam) : nullptr;
    if (!f) {
        g_err = "lam not factored";
        return HEVI_ENOFACTOR;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const size_t bytes = sizeof(double) * pl->g.Z * pl->g.Z;
    if (A_host) CK(cudaMemcpyAsync(A_host, f->A, bytes, cudaMemcpyDeviceToHost, st));
    if (LU_host) CK(cudaMemcpyAsync(LU_host, f->LU, bytes, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return HEVI_OK;
}

// the fused step chains P' of the stage-0 input through stage 2 of the
// previous step (explicit_col M_S3 writes P'(Q^{n+1}) into work's Q1 field 0)
static bool pp_chainable(const hevi_plan* pl) {
    const Geo& g = pl->g;
    return pl->use_col && pl->use_v2 && pl->use_tma && pl->lt_ok && pl->eqset == 0 && pl->N == 4 &&
           pl->Ny == 4 && !g.slab && (g.x0 % 2) == 0 && (g.px % 2) == 0;
}

int hevi_rhs(hevi_plan* pl, const double* q, double* R, void* stream) {
    if (!pl || !q || !R) return fail("null argument");
    EArgs a = base_eargs(pl);
    a.q = q;
    a.out = R;
    a.stage = 0;
    if (pl->eqset == 0 && pp_chainable(pl)) {
        // the production column sweep reads P'(q) as a plane: form it first
        if (!pl->ppscratch) CK(cudaMalloc(&pl->ppscratch, sizeof(double) * pl->g.fs));
        BC16 bcv;
        memcpy(bcv.v, pl->bc, sizeof(bcv.v));
        const dim3 grid((pl->g.lX + 255) / 256, pl->g.lY, pl->g.Z);
        k_pp_plane<<<grid, 256, 0, (cudaStream_t)stream>>>(pl->g, pl->lv, pl->ph, q, pl->ppscratch, bcv);
        CK(cudaGetLastError());
        a.pp_in = pl->ppscratch;
    }
    return run_e(pl, M_R, a, (cudaStream_t)stream);
}

int hevi_linear_v(hevi_plan* pl, const double* q, double* L, void* stream) {
    if (!pl || !q || !L) return fail("null argument");
    EArgs a = base_eargs(pl);
    a.q = q;
    a.out = L;
    return run_e(pl, M_L, a, (cudaStream_t)stream);
}

int hevi_solve(hevi_plan* pl, double lam, const double* qe, double* q, void* stream) {
    if (!pl || !qe || !q) return fail("null argument");
    if (!(lam > 0.0)) return fail("implicit solve requires positive lam");
    int rc = hevi_factor(pl, lam, nullptr, stream);
    if (rc) return rc;
    SArgs a = base_sargs(pl, find_factor(pl, lam));
    a.P = qe;
    a.out = q;
    a.src_uv = qe;
    return run_s(pl, a, (cudaStream_t)stream);
}

int hevi_pp_refresh(hevi_plan* pl, const double* Q, double* work, void* stream) {
    if (!pl || !Q || !work) return fail("null argument");
    if (pl->eqset != 0) return HEVI_OK;
    BC16 bcv;
    memcpy(bcv.v, pl->bc, sizeof(bcv.v));
    const dim3 grid((pl->g.lX + 255) / 256, pl->g.lY, pl->g.Z);
    k_pp_plane<<<grid, 256, 0, (cudaStream_t)stream>>>(pl->g, pl->lv, pl->ph, Q, work, bcv);
    CK(cudaGetLastError());
    return HEVI_OK;
}

static int stage_impl(hevi_plan* pl, int stage, double dt, const double* tab, double* Q, double* work,
                      bool pp_chain, void* stream, int tmode = 0) {
    if (!pl || !tab || !Q || !work) return fail("null argument");
    const long long fs5 = 5 * pl->g.fs;
    double* Q1 = work;
    double* A = work + fs5;
    double* F = work + 2 * fs5;
    double* P = work + 3 * fs5;
    const double* a_ = tab;        // a[3][3]
    const double* at = tab + 9;    // at[3][3]
    const double* b = tab + 18;    // b[3]
    EArgs a = base_eargs(pl);
    a.dt = dt;
    a.stage = stage;
    a.tmode = tmode;
    int mode;
    if (stage == 0) {
        mode = M_S1;
        pl->pp_ok[0] = pl->pp_ok[1] = 0;   // a new step: the solves will refill the P' planes
        // split stage (tmode != 0) without the chain: both calls form P'(Q) over
        // the window, the boundary call after the exchange refreshed the halos
        if (pl->eqset == 0 && pl->use_v2) {
            // P'(Q) into Q1 field 0: not written by stage 0 (it writes Q1 u, v),
            // overwritten by the stage-0 solve afterwards; with pp_chain the
            // previous step's stage 2 already wrote it there
            if (!pp_chain) {
                int rc = hevi_pp_refresh(pl, Q, Q1, stream);
                if (rc) return rc;
            }
            a.pp_in = Q1;
        }
        a.q = Q;
        a.P = P;
        a.Quv = Q1;
        a.A = A;
        a.F = F;
        a.a_p = a_[3 * 1 + 0];
        a.at_p = at[3 * 1 + 0];
        a.a_a = a_[3 * 2 + 0];
        a.at_a = at[3 * 2 + 0];
        a.cb = dt * b[0];
    } else if (stage == 1) {
        mode = M_S2;
        a.q = Q1;
        a.P = P;
        a.Quv = A;
        a.A = A;
        a.F = F;
        if (pl->pp_ok[0] && pl->pp_work == work) a.pp_in = P + pl->g.fs;
        a.a_p = a_[3 * 2 + 1];
        a.at_p = at[3 * 2 + 1];
        a.cb = dt * b[1];
    } else if (stage == 2) {
        mode = M_S3;
        a.q = A;
        a.F = F;
        a.out = Q;
        if (pl->pp_ok[1] && pl->pp_work == work) a.pp_in = P + 2 * pl->g.fs;
        // Q1 is dead after stage 1: its field 0 takes P'(Q^{n+1}) (explicit_col only)
        a.pp_out = Q1;
        a.cb = dt * b[2];
    } else {
        return fail("stage must be 0, 1 or 2");
    }
    return run_e(pl, mode, a, (cudaStream_t)stream);
}

int hevi_stage(hevi_plan* pl, int stage, double dt, const double* tab, double* Q, double* work,
               void* stream) {
    return stage_impl(pl, stage, dt, tab, Q, work, false, stream);
}

int hevi_stage_ex(hevi_plan* pl, int stage, double dt, const double* tab, double* Q, double* work,
                  unsigned flags, void* stream) {
    const bool chain = stage == 0 && (flags & HEVI_STEP_PP_VALID) && pl && pp_chainable(pl);
    if ((flags & HEVI_STAGE_INTERIOR) && (flags & HEVI_STAGE_BOUNDARY))
        return fail("HEVI_STAGE_INTERIOR and HEVI_STAGE_BOUNDARY are exclusive");
    const int tmode = (flags & HEVI_STAGE_INTERIOR) ? 1 : (flags & HEVI_STAGE_BOUNDARY) ? 2 : 0;
    return stage_impl(pl, stage, dt, tab, Q, work, chain, stream, tmode);
}

int hevi_stage_tiles(const hevi_plan* pl, int* n_interior, int* n_boundary) {
    if (!pl || !n_interior || !n_boundary) return fail("null argument");
    int tb[6];
    tile_split(pl->g, 4, HEVI_ECOL_TY, tb);
    *n_interior = (tb[3] - tb[2]) * (tb[5] - tb[4]);
    *n_boundary = tb[0] * tb[1] - *n_interior;
    return HEVI_OK;
}

int hevi_stage_solve(hevi_plan* pl, int stage, double lam, double* work, void* stream) {
    if (!pl || !work) return fail("null argument");
    const Factor* f = find_factor(pl, lam);
    if (!f) {
        g_err = "lam not factored (call hevi_factor first)";
        return HEVI_ENOFACTOR;
    }
    if (stage != 0 && stage != 1) return fail("stage must be 0 or 1");
    const long long fs5 = 5 * pl->g.fs;
    SArgs a = base_sargs(pl, f);
    a.P = work + 3 * fs5;
    a.out = stage == 0 ? work : work + fs5;
    a.src_uv = nullptr;
    // set2nc: P' of the solved stage state into field 1 + stage of the P buffer
    a.pp_out = pl->eqset == 0 ? work + 3 * fs5 + (1 + stage) * pl->g.fs : nullptr;
    memcpy(a.bc, pl->bc, sizeof(a.bc));
    bool v2 = false;
    const int rc = run_s(pl, a, (cudaStream_t)stream, &v2);
    pl->pp_ok[stage] = (rc == HEVI_OK && v2 && a.pp_out) ? 1 : 0;
    pl->pp_work = work;
    return rc;
}

int hevi_ark2_step_ex(hevi_plan* pl, double dt, const double* tab, double* Q, double* work,
                      unsigned flags, void* stream) {
    if (!pl || !tab) return fail("null argument");
    const double lam = tab[9 + 3 * 1 + 1] * dt;  // problem.lam = tableau.diag * dt
    int rc = hevi_factor(pl, lam, nullptr, stream);
    if (rc) return rc;
    const bool chain = (flags & HEVI_STEP_PP_VALID) && pp_chainable(pl);
    if ((rc = stage_impl(pl, 0, dt, tab, Q, work, chain, stream))) return rc;
    if ((rc = hevi_stage_solve(pl, 0, lam, work, stream))) return rc;
    if ((rc = stage_impl(pl, 1, dt, tab, Q, work, false, stream))) return rc;
    if ((rc = hevi_stage_solve(pl, 1, lam, work, stream))) return rc;
    return stage_impl(pl, 2, dt, tab, Q, work, false, stream);
}

int hevi_ark2_step(hevi_plan* pl, double dt, const double* tab, double* Q, double* work,
                   void* stream) {
    return hevi_ark2_step_ex(pl, dt, tab, Q, work, 0u, stream);
}

int hevi_step_chains_pp(const hevi_plan* pl) { return pl && pp_chainable(pl) ? 1 : 0; }

int hevi_rk35_step(hevi_plan* pl, double dt, double* Q, double* work, void* stream) {
    if (!pl || !Q || !work) return fail("null argument");
    // Shu-Osher coefficients of SSP RK(5,3) (imexcore.py:81-94): stage i combines
    // alpha_a u_a (optional), alpha_b u_{i-1} and beta dt R(u_{i-1})
    static const double al_a[5] = {0.0, 0.0, 0.355909775063327, 0.367933791638137,
                                   0.237593836598569};
    static const double al_b[5] = {1.0, 1.0, 0.644090224936674, 0.632066208361863,
                                   0.762406163401431};
    static const double be[5] = {0.377268915331368, 0.377268915331368, 0.242995220537396,
                                 0.238458932846290, 0.287632146308408};
    const long long fs5 = 5 * pl->g.fs;
    double* W[4] = {work, work + fs5, work + 2 * fs5, work + 3 * fs5};
    double* qin[5] = {Q, W[0], W[1], W[2], W[3]};
    double* xin[5] = {nullptr, nullptr, Q, Q, W[1]};
    double* out[5] = {W[0], W[1], W[2], W[3], Q};
    for (int i = 0; i < 5; ++i) {
        EArgs a = base_eargs(pl);
        a.q = qin[i];
        a.A = xin[i];
        a.out = out[i];
        a.a_p = al_a[i];
        a.at_p = al_b[i];
        a.cb = be[i] * dt;
        a.stage = i < 2 ? i : 2;
        a.rk_final = (i == 4);
        int rc = run_e(pl, M_RK, a, (cudaStream_t)stream);
        if (rc) return rc;
    }
    return HEVI_OK;
}

int hevi_evec_to_lattice(hevi_plan* pl, const double* E, double* Lt, int nf, void* stream) {
    if (!pl || !E || !Lt) return fail("null argument");
    CArgs a;
    a.g = pl->g;
    a.N = pl->N;
    a.Ny = pl->Ny;
    a.nel = (long long)pl->g.nex * pl->g.ney * pl->g.nez;
    const long long n = (long long)pl->g.lX * pl->g.lY * pl->g.Z;
    k_e2l<<<blocks_for(n), 256, 0, (cudaStream_t)stream>>>(E, Lt, a, nf);
    CK(cudaGetLastError());
    return HEVI_OK;
}

int hevi_dss(hevi_plan* pl, const double* Ein, double* Eout, int nf, const double* wx, const double* wy,
             const double* wz, void* stream) {
    if (!pl || !Ein || !Eout || !wx || !wy || !wz) return fail("null argument");
    if (pl->g.lX != pl->g.X || pl->g.lY != pl->g.Y) return fail("hevi_dss needs a whole-domain plan");
    if (Ein == Eout) return fail("hevi_dss: input and output must not alias");
    CArgs a;
    a.g = pl->g;
    a.N = pl->N;
    a.Ny = pl->Ny;
    a.nel = (long long)pl->g.nex * pl->g.ney * pl->g.nez;
    const long long n = (long long)pl->g.X * pl->g.Y * pl->g.Z;
    k_dss<<<blocks_for(n), 256, 0, (cudaStream_t)stream>>>(Ein, Eout, a, nf, wx, wy, wz);
    CK(cudaGetLastError());
    return HEVI_OK;
}

int hevi_lattice_to_evec(hevi_plan* pl, const double* Lt, double* E, int nf, void* stream) {
    if (!pl || !E || !Lt) return fail("null argument");
    if (pl->g.lX != pl->g.X || pl->g.lY != pl->g.Y) return fail("lattice_to_evec needs the full lattice");
    CArgs a;
    a.g = pl->g;
    a.N = pl->N;
    a.Ny = pl->Ny;
    a.nel = (long long)pl->g.nex * pl->g.ney * pl->g.nez;
    const long long n = a.nel * (pl->N + 1) * (pl->Ny + 1) * (pl->N + 1);
    k_l2e<<<blocks_for(n), 256, 0, (cudaStream_t)stream>>>(Lt, E, a, nf);
    CK(cudaGetLastError());
    return HEVI_OK;
}

int hevi_flags(hevi_plan* pl, unsigned* flags, int reset, void* stream) {
    if (!pl || !flags) return fail("null argument");
    cudaStream_t st = (cudaStream_t)stream;
    CK(cudaMemcpyAsync(pl->h_flags, pl->d_flags, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    if (reset) CK(cudaMemsetAsync(pl->d_flags, 0, sizeof(unsigned), st));
    CK(cudaStreamSynchronize(st));
    *flags = pl->h_flags[0];
    return HEVI_OK;
}

int hevi_band_pack(const double* dense, double* band, int n_col, int M, int nb, void* stream) {
    if (!dense || !band || n_col < 1 || M < 1 || nb < 1) return fail("bad band_pack arguments");
    k_band_pack<<<blocks_for((long long)n_col * M * (2 * nb - 1)), 256, 0, (cudaStream_t)stream>>>(
        dense, band, n_col, M, nb);
    CK(cudaGetLastError());
    return HEVI_OK;
}

int hevi_band_unpack(const double* band, double* dense, int n_col, int M, int nb, void* stream) {
    if (!dense || !band || n_col < 1 || M < 1 || nb < 1) return fail("bad band_unpack arguments");
    k_band_unpack<<<blocks_for((long long)n_col * M * M), 256, 0, (cudaStream_t)stream>>>(
        band, dense, n_col, M, nb);
    CK(cudaGetLastError());
    return HEVI_OK;
}

int hevi_band_lu(double* band, int n_col, int M, int nb, double norm, int* bad_col, void* stream) {
    if (!band || !bad_col || n_col < 1 || M < 1 || nb < 1) return fail("bad band_lu arguments");
    cudaStream_t st = (cudaStream_t)stream;
    int* d_bad;
    CK(cudaMallocAsync(&d_bad, sizeof(int), st));
    const int big = 0x7fffffff;
    CK(cudaMemcpyAsync(d_bad, &big, sizeof(int), cudaMemcpyHostToDevice, st));
    k_band_lu<<<(n_col + 127) / 128, 128, 0, st>>>(band, n_col, M, nb, norm, d_bad);
    CK(cudaGetLastError());
    int h = big;
    CK(cudaMemcpyAsync(&h, d_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(d_bad, st));
    CK(cudaStreamSynchronize(st));
    *bad_col = (h == big) ? -1 : h;
    return HEVI_OK;
}

int hevi_band_solve(const double* band, double* rhs, int n_col, int M, int nb, void* stream) {
    if (!band || !rhs || n_col < 1 || M < 1 || nb < 1) return fail("bad band_solve arguments");
    k_band_solve<<<(n_col + 127) / 128, 128, 0, (cudaStream_t)stream>>>(band, rhs, n_col, M, nb);
    CK(cudaGetLastError());
    return HEVI_OK;
}

// ---- 3D-IMEX operators (imex3d.cuh) ----------------------------------------
static I3Args i3args(const hevi_plan* pl, double lam) {
    I3Args a;
    a.g = pl->g;
    a.lv = pl->lv;
    a.ph = pl->ph;
    a.cx = pl->cx;
    a.cy = pl->cy;
    a.cz = pl->cz;
    a.Dx = pl->Dx;
    a.Dy = pl->Dy;
    a.Dz = pl->Dz;
    a.N = pl->N;
    a.Ny = pl->Ny;
    a.eqset = pl->eqset;
    a.ainv_identity = pl->ainv_identity;
    a.vert_only = 0;
    a.lam = lam;
    return a;
}

static int i3blocks(const hevi_plan* pl) {
    const long long n = (long long)pl->g.Z * pl->g.lY * pl->g.lX;
    return (int)((n + 255) / 256);
}

int hevi_linear3(hevi_plan* pl, const double* q, double* out, void* stream) {
    if (!pl || !q || !out) return fail("null argument");
    k3_linear<<<i3blocks(pl), 256, 0, (cudaStream_t)stream>>>(i3args(pl, 0.0), q, out);
    CK(cudaGetLastError());
    return HEVI_OK;
}

int hevi_grad(hevi_plan* pl, int vertical_only, const double* f, double* out, void* stream) {
    if (!pl || !f || !out) return fail("null argument");
    I3Args a = i3args(pl, 0.0);
    a.vert_only = vertical_only ? 1 : 0;
    k3_grad<<<i3blocks(pl), 256, 0, (cudaStream_t)stream>>>(a, f, out);
    CK(cudaGetLastError());
    return HEVI_OK;
}

int hevi_div(hevi_plan* pl, int vertical_only, const double* vec, double* out, void* stream) {
    if (!pl || !vec || !out) return fail("null argument");
    I3Args a = i3args(pl, 0.0);
    a.vert_only = vertical_only ? 1 : 0;
    k3_div<<<i3blocks(pl), 256, 0, (cudaStream_t)stream>>>(a, vec, out);
    CK(cudaGetLastError());
    return HEVI_OK;
}

int hevi_schur3_up(hevi_plan* pl, double lam, int vertical_only, const double* P, double* up,
                   void* stream) {
    if (!pl || !P || !up) return fail("null argument");
    I3Args a = i3args(pl, lam);
    a.vert_only = vertical_only != 0;
    k3_up<<<i3blocks(pl), 256, 0, (cudaStream_t)stream>>>(a, P, up);
    CK(cudaGetLastError());
    return HEVI_OK;
}

int hevi_schur3_flux(hevi_plan* pl, double lam, int vertical_only, const double* P, const double* vel,
                     double* out, void* stream) {
    if (!pl || !P || !vel || !out) return fail("null argument");
    I3Args a = i3args(pl, lam);
    a.vert_only = vertical_only != 0;
    k3_flux<<<i3blocks(pl), 256, 0, (cudaStream_t)stream>>>(a, P, vel, out);
    CK(cudaGetLastError());
    return HEVI_OK;
}

int hevi_schur3_ua(hevi_plan* pl, double lam, const double* qe, double* ua, double* Pe, void* stream) {
    if (!pl || !qe || !ua || !Pe) return fail("null argument");
    k3_ua<<<i3blocks(pl), 256, 0, (cudaStream_t)stream>>>(i3args(pl, lam), qe, ua, Pe);
    CK(cudaGetLastError());
    return HEVI_OK;
}

int hevi_schur3_extract(hevi_plan* pl, double lam, const double* P, const double* ua,
                        const double* up, const double* qe, double* q, void* stream) {
    if (!pl || !P || !ua || !up || !qe || !q) return fail("null argument");
    k3_extract<<<i3blocks(pl), 256, 0, (cudaStream_t)stream>>>(i3args(pl, lam), P, ua, up, qe, q);
    CK(cudaGetLastError());
    return HEVI_OK;
}

int hevi_wdot(const hevi_plan* pl, const double* x, const double* y, int nf, double* out_host,
              void* stream) {
    if (!pl || !x || !y || !out_host || nf < 1) return fail("bad wdot arguments");
    cudaStream_t st = (cudaStream_t)stream;
    double* d;
    CK(cudaMallocAsync(&d, sizeof(double) * (KV_BLOCKS + 1), st));
    k3_wdot<<<KV_BLOCKS, KV_T, 0, st>>>(pl->g, pl->N, pl->Ny, nf, x, y, d);
    CK(cudaGetLastError());
    k3_sum<<<1, 32, 0, st>>>(d, KV_BLOCKS, d + KV_BLOCKS);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out_host, d + KV_BLOCKS, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(d, st));
    CK(cudaStreamSynchronize(st));
    return HEVI_OK;
}

int hevi_axpby(long long n, double alpha, const double* x, double beta, double* y, void* stream) {
    if (!x || !y || n < 0) return fail("bad axpby arguments");
    if (n == 0) return HEVI_OK;
    const long long b = (n + 255) / 256;
    k3_axpby<<<(int)(b < 1184 ? b : 1184), 256, 0, (cudaStream_t)stream>>>(n, alpha, x, beta, y);
    CK(cudaGetLastError());
    return HEVI_OK;
}

int hevi_plan_set_option(hevi_plan* pl, int option, int value) {
    if (!pl) return fail("null plan");
    if (option == HEVI_OPT_FORCE_PIVOTED) {
        pl->force_pivoted = value != 0;
        return HEVI_OK;
    }
    return fail("unknown plan option");
}

int hevi_factor_pivoted(const hevi_plan* pl, double lam, int* pivoted) {
    const Factor* f = pl ? find_factor(pl, lam) : nullptr;
    if (!f) {
        g_err = "lam not factored";
        return HEVI_ENOFACTOR;
    }
    if (pivoted) *pivoted = f->pivoted;
    return HEVI_OK;
}

int hevi_lu_pivot(double* A, int* piv, int n_col, int M, int* info_host, void* stream) {
    if (!A || !piv || n_col < 1 || M < 1) return fail("bad lu_pivot arguments");
    cudaStream_t st = (cudaStream_t)stream;
    int* d_info;
    CK(cudaMallocAsync(&d_info, sizeof(int) * n_col, st));
    k_lu_pivot_batched<<<n_col, 256, 0, st>>>(A, piv, M, d_info);
    CK(cudaGetLastError());
    if (info_host) CK(cudaMemcpyAsync(info_host, d_info, sizeof(int) * n_col, cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(d_info, st));
    CK(cudaStreamSynchronize(st));
    return HEVI_OK;
}

int hevi_lu_pivot_solve(const double* LU, const int* piv, double* rhs, int n_col, int M, void* stream) {
    if (!LU || !piv || !rhs || n_col < 1 || M < 1) return fail("bad lu_pivot_solve arguments");
    k_lu_pivot_solve<<<(n_col + 127) / 128, 128, 0, (cudaStream_t)stream>>>(LU, piv, rhs, n_col, M);
    CK(cudaGetLastError());
    return HEVI_OK;
}

int hevi_diagnostics(const hevi_plan* pl, const double* q, const double* wx, const double* wy,
                     const double* wz, double* out_host, void* stream) {
    if (!pl || !q || !wx || !wy || !wz || !out_host) return fail("null argument");
    cudaStream_t st = (cudaStream_t)stream;
    double* d;
    CK(cudaMallocAsync(&d, sizeof(double) * (3 * DIAG_BLOCKS + 3), st));
    k_diag_partial<<<DIAG_BLOCKS, DIAG_T, 0, st>>>(pl->g, q, pl->lv.rho0, wx, wy, wz, d);
    CK(cudaGetLastError());
    k_diag_final<<<1, 32, 0, st>>>(d, d + 3 * DIAG_BLOCKS);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out_host, d + 3 * DIAG_BLOCKS, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(d, st));
    CK(cudaStreamSynchronize(st));
    return HEVI_OK;
}

int hevi_std_solve(const hevi_plan* pl, const double* band, int M, int nb, const double* qe, double* q,
                   void* stream) {
    if (!pl || !band || !qe || !q || nb < 1 || M != 5 * pl->g.Z) return fail("bad std_solve arguments");
    const Geo& g = pl->g;
    const size_t smem = sizeof(double) * (size_t)(2 * nb - 1) * M;
    if (smem > 225 * 1024) return fail("standard-form band too wide for the column kernel");
    CK(cudaFuncSetAttribute(k_std_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int NYo = g.slab ? 1 : pl->N;
    const long long nc = ((long long)(g.ex_e - g.ex_b) * pl->N + (g.ex_e == g.nex ? 1 : 0)) *
                         ((long long)(g.ey_e - g.ey_b) * NYo + (g.ey_e == g.ney ? 1 : 0));
    k_std_solve<<<(int)((nc + 127) / 128), 128, smem, (cudaStream_t)stream>>>(g, pl->N, band, M, nb, qe, q);
    CK(cudaGetLastError());
    return HEVI_OK;
}

static int halo_call(const hevi_plan* pl, double* q, int nf, int xlo, int xhi, int ylo, int yhi,
                     double* buf, int unpack, void* stream) {
    if (!pl || !q || !buf || nf < 1) return fail("null argument");
    const Geo& g = pl->g;
    if (xlo < g.x0 || xhi > g.x0 + g.lX || ylo < g.y0 || yhi > g.y0 + g.lY || xlo >= xhi || ylo >= yhi)
        return fail("halo region outside the plan's window");
    const long long n = (long long)nf * g.Z * (yhi - ylo) * (xhi - xlo);
    k_halo<<<blocks_for(n), 256, 0, (cudaStream_t)stream>>>(g, q, nf, xlo, xhi, ylo, yhi, buf, unpack);
    CK(cudaGetLastError());
    return HEVI_OK;
}

int hevi_halo_pack(const hevi_plan* pl, const double* q, int nf, int xlo, int xhi, int ylo, int yhi,
                   double* buf, void* stream) {
    return halo_call(pl, const_cast<double*>(q), nf, xlo, xhi, ylo, yhi, buf, 0, stream);
}

int hevi_halo_unpack(const hevi_plan* pl, double* q, int nf, int xlo, int xhi, int ylo, int yhi,
                     const double* buf, void* stream) {
    return halo_call(pl, q, nf, xlo, xhi, ylo, yhi, const_cast<double*>(buf), 1, stream);
}

int hevi_absmax(const double* a, long long n, double* out_host, void* stream) {
    if (!a || !out_host) return fail("null argument");
    cudaStream_t st = (cudaStream_t)stream;
    unsigned long long* d;
    CK(cudaMallocAsync(&d, sizeof(unsigned long long), st));
    CK(cudaMemsetAsync(d, 0, sizeof(unsigned long long), st));
    k_absmax<<<blocks_for(n), 256, 0, st>>>(a, n, d);
    CK(cudaGetLastError());
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(d, st));
    CK(cudaStreamSynchronize(st));
    double v;
    memcpy(&v, &h, sizeof(v));
    *out_host = v;
    return HEVI_OK;
}

#include "general_api.cuh"

}  // extern "C"
