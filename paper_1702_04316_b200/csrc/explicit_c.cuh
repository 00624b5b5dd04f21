// explicit_c.cuh -- explicit-stage kernel for the conservative equation set
// ``set2c`` (included by hevi.cu inside its anonymous namespace).
//
// euler.nonlinear_rhs set2c (euler.py:474-487) is a flux form,
//   R = -( div U,  div(U_m U / rho + P' e_m) + rho' g e_z,  div(theta U) ),
// so with the DSS folded into the derivatives (see hevi.cu) each point needs
// the x-, y- and z-derivatives of 12 pointwise flux fields.  The element layer
// staged in shared memory therefore carries the fluxes themselves:
//   0 U, 1 V, 2 W, 3 UU/rho+P', 4 VV/rho+P', 5 WW/rho+P', 6 UV/rho, 7 UW/rho,
//   8 VW/rho, 9 theta U, 10 theta V, 11 theta W, 12 F0 Theta' (linearised
//   pressure, euler.py:192-193), 13 rho', 14 Theta'.
// One thread per owned point (the v1 structure: per-point derivative lines,
// sweep over element layers with the z-face carry in shared memory).  The
// secondary equation set of the path; set2nc uses the tuned explicit_v2.
#pragma once

// P' = EOS(rho, theta) - P0f about the background state: Pb (1+delta)^gamma - P0f
// by the binomial series of explicit_v2.cuh (|delta| <= 1/8), exact pow beyond
__device__ __forceinline__ double pprime_delta(double delta, double rho, double theta, double Pb,
                                               double c0, double P0f, const double* bc,
                                               const Phys& ph) {
    if (fabs(delta) <= 0.125) {
        double s = bc[14];
#pragma unroll
        for (int k = 13; k >= 0; --k) s = fma(s, delta, bc[k]);
        return fma(Pb, s * delta, c0);
    }
    return ph.P0 * pow(rho * ph.R * theta / ph.P0, ph.gamma) - P0f;
}

template <int NX, int NY, int TX, int TY>
struct ECT {
    static constexpr int OX = TX * NX, OY = TY * NY;
    static constexpr int LX = OX + NX + 1, LY = OY + NY + 1, LZ = NX + 1;
    static constexpr int PL = LX * LY, VOL = PL * LZ;
    static constexpr int CXW = OX + 1, CYW = OY + 1 + (NY == 1 ? 1 : 0);
    static constexpr int NSF = 15;
    static constexpr int DXS = (NX + 1) * (NX + 1), DYS = (NY + 1) * (NY + 1);
    static constexpr size_t SMEM = sizeof(double) * (size_t)(NSF * VOL + NSF * CXW * CYW + DXS + DYS);
    static constexpr int PTS = OX * (OY + (NY == 1 ? 1 : 0)) * NX;
    static constexpr int BLK0 = PTS < 64 ? 64 : (PTS > 512 ? 512 : PTS);
    static constexpr int BLK = (BLK0 + 31) / 32 * 32;
};

template <int NX, int NY, int TX, int TY, int MODE>
__global__ void __launch_bounds__(ECT<NX, NY, TX, TY>::BLK) k_explicit_c(const EArgs a) {
    using T = ECT<NX, NY, TX, TY>;
    constexpr int NZ = NX;
    constexpr int LX = T::LX, PL = T::PL, VOL = T::VOL, CXW = T::CXW, CYW = T::CYW;
    constexpr int BLK = T::BLK;
    constexpr bool NEED_L = (MODE == M_L || MODE == M_S1 || MODE == M_S2);
    constexpr bool NEED_R = (MODE != M_L);
    extern __shared__ __align__(16) double smc[];
    double* S = smc;
    double* Cr = S + T::NSF * VOL;
    double* sDx = Cr + T::NSF * CXW * CYW;
    double* sDy = sDx + T::DXS;

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

    for (int ez = 0; ez < g.nez; ++ez) {
        const int gz0 = ez * NZ;
        // ---------------- load the layer, form the flux fields --------------
        for (int idx = tid; idx < VOL; idx += BLK) {
            const int lx = idx % LX;
            const int t = idx / LX;
            const int ly = t % T::LY;
            const int lz = t / T::LY;
            const int gx = gxlo + lx, gy = gylo + ly, gz = gz0 + lz;
            const int ix = gx - g.x0, iy = gy - g.y0;
            double f[15];
#pragma unroll
            for (int k = 0; k < 15; ++k) f[k] = 0.0;
            if (gx >= 0 && gx < g.X && gy >= 0 && gy < g.Y && ix >= 0 && ix < g.lX && iy >= 0 &&
                iy < g.lY) {
                const double* qp = a.q + ((long long)gz * g.lY + iy) * g.px + ix;
                const double r = __ldg(qp), U = __ldg(qp + g.fs), V = __ldg(qp + 2 * g.fs),
                             W = __ldg(qp + 3 * g.fs), Th = __ldg(qp + 4 * g.fs);
                f[0] = U;
                f[1] = V;
                f[2] = W;
                f[13] = r;
                f[14] = Th;
                if (NEED_R) {
                    // euler.py:476-480: rho, Theta, theta = Theta / rho, P' = EOS - P0f
                    const double rho = __ldg(a.lv.rho0 + gz) + r;
                    const double Theta = __ldg(a.lv.Th0 + gz) + Th;
                    const double theta = Theta / rho;
                    // P = P0 (rho R theta / P0)^gamma evaluated about the background
                    // (rho theta = Theta): delta = Theta' / Theta0, series as set2nc
                    const double pp = pprime_delta(Th * __ldg(a.lv.iTh0 + gz), rho, theta,
                                                   __ldg(a.lv.E0 + gz), __ldg(a.lv.c0 + gz),
                                                   __ldg(a.lv.P0f + gz), a.bc, a.ph);
                    const double irho = 1.0 / rho;
                    // euler.py:483: Fm = U_m U / rho, Fm[m] += P'
                    f[3] = (U * U) * irho + pp;
                    f[4] = (V * V) * irho + pp;
                    f[5] = (W * W) * irho + pp;
                    f[6] = (U * V) * irho;
                    f[7] = (U * W) * irho;
                    f[8] = (V * W) * irho;
                    // euler.py:487: theta U
                    f[9] = theta * U;
                    f[10] = theta * V;
                    f[11] = theta * W;
                }
                if (NEED_L) f[12] = __ldg(a.lv.F0c + gz) * Th;
            }
#pragma unroll
            for (int k = 0; k < 15; ++k) S[k * VOL + idx] = f[k];
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
            double dxa[NX + 1], dxb[NX + 1], dya[NY + 1], dyb[NY + 1], dza[NZ + 1], dzn[NZ + 1];
#pragma unroll
            for (int m = 0; m <= NX; ++m) {
                dxa[m] = sDx[ax.row * (NX + 1) + m];
                dxb[m] = sDx[NX * (NX + 1) + m];
                dza[m] = sDx[az.row * (NZ + 1) + m];
                dzn[m] = sDx[NZ * (NZ + 1) + m];
            }
#pragma unroll
            for (int m = 0; m <= NY; ++m) {
                dya[m] = sDy[ay.row * (NY + 1) + m];
                dyb[m] = sDy[NY * (NY + 1) + m];
            }
            const int cidx = oy * CXW + ox;
            auto ddx = [&](int f) {
                const double* sx = S + f * VOL + lz * PL + ly * LX;
                double d = dline<NX, 1>(sx + ax.s0, dxa);
                if (ax.face) d += dline<NX, 1>(sx + ax.s1, dxb);
                return cx * d;
            };
            auto ddy = [&](int f) {
                const double* sy = S + f * VOL + lz * PL + lx;
                double e = dline<NY, LX>(sy + ay.s0 * LX, dya);
                if (ay.face) e += dline<NY, LX>(sy + ay.s1 * LX, dyb);
                return cy * e;
            };
            auto ddz = [&](int f) {
                const double* sz = S + f * VOL + ly * LX + lx;
                double d = dline<NZ, PL>(sz + az.s0 * PL, dza);
                if (az.face) d += Cr[f * CXW * CYW + cidx];
                return cz * d;
            };
            const int c0 = lz * PL + ly * LX + lx;
            const double r = S[13 * VOL + c0], U = S[0 * VOL + c0], V = S[1 * VOL + c0],
                         W = S[2 * VOL + c0], Th = S[14 * VOL + c0];
            const bool bx = (gx == 0) || (gx == g.X - 1);
            const bool by = g.slab || (gy == 0) || (gy == g.Y - 1);
            const bool bz = (gz == 0) || (gz == g.Z - 1);
            const double dWz = ddz(2);
            double Rv[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
            if (NEED_R) {
                const double rho = __ldg(a.lv.rho0 + gz) + r;
                const double Theta = __ldg(a.lv.Th0 + gz) + Th;
                if (!(isfinite(r) && isfinite(U) && isfinite(V) && isfinite(W) && isfinite(Th)))
                    atomicOr(a.flags, HEVI_F_NONFINITE_IN(a.stage));
                if (!(rho > 0.0) || !(Theta / rho > 0.0)) atomicOr(a.flags, HEVI_F_EOS(a.stage));
                // euler.nonlinear_rhs set2c (euler.py:481-487), DSS folded into the derivatives
                Rv[0] = -((ddx(0) + ddy(1)) + dWz);
                Rv[1] = -((ddx(3) + ddy(6)) + ddz(7));
                Rv[2] = -((ddx(6) + ddy(4)) + ddz(8));
                Rv[3] = -((ddx(7) + ddy(8)) + ddz(5)) - r * gr;
                Rv[4] = -((ddx(9) + ddy(10)) + ddz(11));
                if (bx) Rv[1] = 0.0;
                if (by) Rv[2] = 0.0;
                if (bz) Rv[3] = 0.0;
            }
            double Lv[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
            if (NEED_L) {
                // euler.linear_operator(vertical_only=True), set2c (euler.py:350-361)
                const double th0 = __ldg(a.lv.theta0 + gz), dth0 = __ldg(a.lv.dth0 + gz);
                Lv[0] = -dWz;
                Lv[3] = bz ? 0.0 : -(ddz(12) + r * gr);
                Lv[4] = -(th0 * dWz + W * dth0);
            }
            // carry: row N of this layer's z-lines (faces of the next layer)
            if (oz == 0 && ez + 1 < g.nez) {
                const int zf[6] = {2, 5, 7, 8, 11, 12};
#pragma unroll
                for (int q = 0; q < 6; ++q) {
                    const double* sz = S + zf[q] * VOL + ly * LX + lx;
                    Cr[zf[q] * CXW * CYW + cidx] = dline<NZ, PL>(sz, dzn);
                }
            }
            const long long o = loff(g, gx, gy, gz);
            const long long fs = g.fs;
            const double qv[5] = {r, U, V, W, Th};
            if (MODE == M_R) {
#pragma unroll
                for (int f = 0; f < 5; ++f) a.out[o + f * fs] = Rv[f];
            } else if (MODE == M_L) {
#pragma unroll
                for (int f = 0; f < 5; ++f) a.out[o + f * fs] = Lv[f];
            } else if (MODE == M_S1) {
                const double dt = a.dt;
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
                    pr[f] = a.A[o + f * fs] + dt * (a.a_p * (Rv[f] - Lv[f]) + a.at_p * Lv[f]);
                    a.F[o + f * fs] = a.F[o + f * fs] + a.cb * Rv[f];
                }
                a.P[o] = pr[0];
                a.P[o + 3 * fs] = pr[3];
                a.P[o + 4 * fs] = pr[4];
                a.Quv[o + fs] = bx ? 0.0 : pr[1];
                a.Quv[o + 2 * fs] = by ? 0.0 : pr[2];
            } else if (MODE == M_RK) {
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
            } else {
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
