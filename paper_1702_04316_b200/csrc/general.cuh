// general.cuh -- the HEVI path on general curvilinear element meshes (the
// cubed-sphere shell), included by hevi.cu inside its
// anonymous namespace.
//
// The box path folds the DSS into a structured unique-point lattice; a
// curvilinear mesh has no such lattice (the panels of the cube meet at edges
// and corners), so this path works on the reference's own E-vector layout
// (nf, nel, nqt, nqs, nqr) with per-node metric terms, exactly the data the
// reference's operators read (specgrid.py:404-455):
//   * element kernels: one CTA per element, one thread per node, the
//     element's fields staged in shared memory, the three reference-direction
//     line sums from there, contracted with the node's contravariant vectors
//     a_r, a_s, a_t (specgrid.grad / div / deriv_vertical, :600-627);
//   * DSS: the coincidence groups as CSR (members in flat-node order, the
//     reference's bincount summation order), one thread per group, the
//     no-flux projector of the group applied on write (euler.py:218-264);
//   * per-column Schur factors: every column's matrix probed by the vertical
//     lhs_schur on the device (columnsolve.py:75-108), batched banded LU
//     with the pivoted dense fallback (:111-153); the solve gathers the
//     Schur RHS into (n_col, M), substitutes per column and scatters back
//     (:191-210).
#pragma once

struct GGeo {
    int nel, nq, NP;           // NP = nq^3 nodes per element
    long long nn;              // nodes
    const double* D;           // nq x nq LGL derivative, row-major
    const double *ar, *as, *at;   // contravariant vectors a^r, a^s, a^t: [3][nn] each
    const double* vert;        // radial unit vector [3][nn]
    const double* Jtv;         // a^t . vert [nn] (specgrid.deriv_vertical)
    const int* bslot;          // [nn]: projector of the node's group, or -1
    const double* bproj;       // [nbp][9]
};

struct GRef {
    const double *rho0, *theta0, *P0f;
    const double *grho0, *gth0, *gvec;   // [3][nn]
    const double *G0, *H0, *F0v;         // set2nc: G0, H0 [nn], F0vec [3][nn]
    const double *Th0, *F0c;             // set2c: Theta0 = rho0 theta0, F0_c [nn]
    const double *Pb, *c0, *irt0;        // EOS(rho0, theta0), Pb - P0f, 1 / (rho0 theta0)
    double g, R, P0, gamma;
    int eqset;                           // 0 set2nc, 1 set2c
    int w_zero;                          // grad theta0 == 0: A^-1 is the identity (imexcore.py:203-206)
    double bc[16];
};

// P' = EOS - P0f at a node without the cancellation (binomial series in
// delta = (rho theta - rho0 theta0) / (rho0 theta0), the box path's pprime)
__device__ __forceinline__ double g_pprime(const GRef& r, long long n, double rho, double dprod) {
    // dprod = rho theta - rho0 theta0  (set2c: Theta')
    const double delta = dprod * r.irt0[n];
    if (fabs(delta) <= 0.125) {
        double s = r.bc[14];
#pragma unroll
        for (int k = 13; k >= 0; --k) s = fma(s, delta, r.bc[k]);
        return fma(r.Pb[n], s * delta, r.c0[n]);
    }
    const double theta = (r.rho0[n] * r.theta0[n] + dprod) / rho;
    return r.P0 * pow(rho * r.R * theta / r.P0, r.gamma) - r.P0f[n];
}

// line sums of a staged element field s at node (i, j, k): d/dr, d/ds, d/dt
// (specgrid.deriv_r / deriv_s / deriv_t, :390-401)
template <int NQ>
__device__ __forceinline__ void g_d3(const double* s, const double* D, int i, int j, int k, double& fr,
                                     double& fs, double& ft) {
    double a = 0.0, b = 0.0, c = 0.0;
#pragma unroll
    for (int m = 0; m < NQ; ++m) {
        a = fma(D[i * NQ + m], s[(k * NQ + j) * NQ + m], a);
        b = fma(D[j * NQ + m], s[(k * NQ + m) * NQ + i], b);
        c = fma(D[k * NQ + m], s[(m * NQ + j) * NQ + i], c);
    }
    fr = a;
    fs = b;
    ft = c;
}

template <int NQ>
__device__ __forceinline__ double g_dt(const double* s, const double* D, int i, int j, int k) {
    double c = 0.0;
#pragma unroll
    for (int m = 0; m < NQ; ++m) c = fma(D[k * NQ + m], s[(m * NQ + j) * NQ + i], c);
    return c;
}

// gradient component c (specgrid.grad: fr a^r + fs a^s + ft a^t)
__device__ __forceinline__ double g_gc(const GGeo& g, long long n, int c, double fr, double fs, double ft) {
    const long long o = c * g.nn + n;
    return (fr * g.ar[o] + fs * g.as[o]) + ft * g.at[o];
}

__device__ __forceinline__ double dot3(const double* a, long long nn, long long n, double x, double y, double z) {
    return (a[n] * x + a[nn + n] * y) + a[2 * nn + n] * z;
}

// the group's no-flux projector on a velocity-like vector (euler.py:261-264)
__device__ __forceinline__ void g_project(const GGeo& g, int slot, double& x, double& y, double& z) {
    if (slot < 0) return;
    const double* P = g.bproj + 9 * (long long)slot;
    const double a = (P[0] * x + P[1] * y) + P[2] * z;
    const double b = (P[3] * x + P[4] * y) + P[5] * z;
    const double c = (P[6] * x + P[7] * y) + P[8] * z;
    x = a;
    y = b;
    z = c;
}

// ---------------------------------------------------------------------------
// R(q) before DSS (euler.py:438-491), one CTA per element
// ---------------------------------------------------------------------------
template <int NQ>
__global__ void __launch_bounds__(NQ * NQ * NQ) kg_rhs(const GGeo g, const GRef r, const double* __restrict__ q,
                                                       double* __restrict__ out, unsigned* flags, int stage) {
    constexpr int NP = NQ * NQ * NQ;
    extern __shared__ double gs[];   // set2nc: 6 planes; set2c: 15
    __shared__ double sD[NQ * NQ];
    const int t = threadIdx.x;
    const long long n = (long long)blockIdx.x * NP + t;
    const long long nn = g.nn;
    for (int i = t; i < NQ * NQ; i += NP) sD[i] = g.D[i];
    const double q0 = q[n], q1 = q[nn + n], q2 = q[2 * nn + n], q3 = q[3 * nn + n], q4 = q[4 * nn + n];
    const double z = fma(q0, 0.0, fma(q1, 0.0, fma(q2, 0.0, fma(q3, 0.0, q4 * 0.0))));
    if (z != z) atomicOr(flags, HEVI_F_NONFINITE_IN(stage));
    const double rho = r.rho0[n] + q0;
    if (r.eqset == 0) {
        const double theta = r.theta0[n] + q4;
        if (!(rho > 0.0) || !(theta > 0.0)) atomicOr(flags, HEVI_F_EOS(stage));
        const double dprod = q0 * r.theta0[n] + q4 * rho;   // rho theta - rho0 theta0
        gs[t] = q0;
        gs[NP + t] = q1;
        gs[2 * NP + t] = q2;
        gs[3 * NP + t] = q3;
        gs[4 * NP + t] = q4;
        gs[5 * NP + t] = g_pprime(r, n, rho, dprod);
    } else {
        const double Theta = r.Th0[n] + q4;
        const double theta = Theta / rho;
        if (!(rho > 0.0) || !(theta > 0.0)) atomicOr(flags, HEVI_F_EOS(stage));
        const double pp = g_pprime(r, n, rho, q4);
        const double U[3] = {q1, q2, q3};
#pragma unroll
        for (int c = 0; c < 3; ++c) gs[c * NP + t] = U[c];
#pragma unroll
        for (int m = 0; m < 3; ++m)
#pragma unroll
            for (int c = 0; c < 3; ++c) gs[(3 + 3 * m + c) * NP + t] = (U[m] * U[c]) / rho + (m == c ? pp : 0.0);
#pragma unroll
        for (int c = 0; c < 3; ++c) gs[(12 + c) * NP + t] = theta * U[c];
    }
    __syncthreads();
    const int i = t % NQ, j = (t / NQ) % NQ, k = t / (NQ * NQ);
    double fr, fs, ft;
    if (r.eqset == 0) {
        const double u[3] = {q1, q2, q3};
        double gr_[6][3];
        double divu = 0.0;
#pragma unroll
        for (int f = 0; f < 6; ++f) {
            g_d3<NQ>(gs + f * NP, sD, i, j, k, fr, fs, ft);
#pragma unroll
            for (int c = 0; c < 3; ++c) gr_[f][c] = g_gc(g, n, c, fr, fs, ft);
            if (f >= 1 && f <= 3) {   // specgrid.div: the m = f-1 terms, r, s, t in order
                const long long o = (f - 1) * nn + n;
                divu = divu + fr * g.ar[o];
                divu = divu + fs * g.as[o];
                divu = divu + ft * g.at[o];
            }
        }
        auto adv = [&](int f) { return (u[0] * gr_[f][0] + u[1] * gr_[f][1]) + u[2] * gr_[f][2]; };
        out[n] = -((adv(0) + dot3(r.grho0, nn, n, u[0], u[1], u[2])) + rho * divu);
#pragma unroll
        for (int c = 0; c < 3; ++c)
            out[(1 + c) * nn + n] = -((adv(1 + c) + gr_[5][c] / rho) + (q0 / rho) * r.gvec[c * nn + n]);
        out[4 * nn + n] = -(adv(4) + dot3(r.gth0, nn, n, u[0], u[1], u[2]));
    } else {
        // div of the vector whose components are planes p0, p0+1, p0+2
        auto divp = [&](int p0) {
            double d = 0.0;
#pragma unroll
            for (int m = 0; m < 3; ++m) {
                g_d3<NQ>(gs + (p0 + m) * NP, sD, i, j, k, fr, fs, ft);
                const long long o = m * nn + n;
                d = d + fr * g.ar[o];
                d = d + fs * g.as[o];
                d = d + ft * g.at[o];
            }
            return d;
        };
        out[n] = -divp(0);
#pragma unroll
        for (int m = 0; m < 3; ++m) out[(1 + m) * nn + n] = -divp(3 + 3 * m) - q0 * r.gvec[m * nn + n];
        out[4 * nn + n] = -divp(12);
    }
}

// ---------------------------------------------------------------------------
// DSS (specgrid.apply_dss, :535-548): the mass-weighted average of every
// coincidence group, summed in flat-node order; with proj the group's
// no-flux projector is applied to fields 1..3 (R: euler.py:493-496)
// ---------------------------------------------------------------------------
__global__ void kg_dss(const int* __restrict__ gptr, const int* __restrict__ gidx, const double* __restrict__ w,
                       const double* __restrict__ wsum, const int* __restrict__ gslot, const double* __restrict__ bproj,
                       const double* in, double* out, int nf, long long nn, int ng, int proj) {
    for (int gi = blockIdx.x * blockDim.x + threadIdx.x; gi < ng; gi += gridDim.x * blockDim.x) {
        const int p0 = gptr[gi], p1 = gptr[gi + 1];
        double v[5];
        for (int f = 0; f < nf; ++f) {
            double num = 0.0;   // np.bincount: w * f summed in flat-node order
            for (int p = p0; p < p1; ++p) {
                const int m = gidx[p];
                num = __dadd_rn(num, __dmul_rn(w[m], in[f * nn + m]));
            }
            const double val = num / wsum[gi];
            if (proj) {
                v[f] = val;
            } else {
                for (int p = p0; p < p1; ++p) out[f * nn + gidx[p]] = val;
            }
        }
        if (proj) {   // nf == 5: the group's projector on the momentum (euler.py:493-496)
            double x = v[1], y = v[2], z = v[3];
            const int s = gslot[gi];
            if (s >= 0) {
                const double* P = bproj + 9 * (long long)s;
                const double a = (P[0] * x + P[1] * y) + P[2] * z;
                const double b = (P[3] * x + P[4] * y) + P[5] * z;
                const double c = (P[6] * x + P[7] * y) + P[8] * z;
                x = a;
                y = b;
                z = c;
            }
            for (int p = p0; p < p1; ++p) {
                const int m = gidx[p];
                out[m] = v[0];
                out[nn + m] = x;
                out[2 * nn + m] = y;
                out[3 * nn + m] = z;
                out[4 * nn + m] = v[4];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// vertical derivatives before DSS: out_p = Jtv * d/dt of a per-node scalar
// (specgrid.deriv_vertical), for up to two scalars formed per node:
//   kind 0: P_lin(q) and q_vel . vert            (vertical_restriction, euler.py:331-337)
//   kind 1: ua . vert  of the Schur RHS velocity (rhs_schur_build, imexcore.py:229-243),
//           ua stored to vec [3][nn]
//   kind 2: a scalar field x (grad_vc(P))
//   kind 3: vec . vert                            (div_vc of a stored vector)
// ---------------------------------------------------------------------------
struct GVArgs {
    const double* q;      // kind 0 / 1: state (5 fields)
    const double* x;      // kind 2: scalar
    double* vec;          // kind 1: ua out; kind 3: vector in
    double* d0;           // first derivative out [nn]
    double* d1;           // second derivative out [nn] (kind 0)
    double lam;
    unsigned* flags;
};

template <int NQ>
__global__ void __launch_bounds__(NQ * NQ * NQ) kg_vderiv(const GGeo g, const GRef r, const GVArgs a, int kind) {
    constexpr int NP = NQ * NQ * NQ;
    __shared__ double s0[NP], s1[NP];
    __shared__ double sD[NQ * NQ];
    const int t = threadIdx.x;
    const long long n = (long long)blockIdx.x * NP + t;
    const long long nn = g.nn;
    for (int i = t; i < NQ * NQ; i += NP) sD[i] = g.D[i];
    const double v0 = g.vert[n], v1 = g.vert[nn + n], v2 = g.vert[2 * nn + n];
    if (kind == 0) {
        const double* q = a.q;
        s0[t] = r.eqset == 0 ? r.G0[n] * q[n] + r.H0[n] * q[4 * nn + n] : r.F0c[n] * q[4 * nn + n];
        s1[t] = (q[nn + n] * v0 + q[2 * nn + n] * v1) + q[3 * nn + n] * v2;
    } else if (kind == 1) {
        const double* q = a.q;
        const double lam = a.lam;
        double x, y, z;
        if (r.eqset == 0) {
            const double coef = (lam * r.H0[n]) / (r.G0[n] * r.rho0[n]);
            const double s = coef * q[4 * nn + n];
            x = q[nn + n] + s * r.gvec[n];
            y = q[2 * nn + n] + s * r.gvec[nn + n];
            z = q[3 * nn + n] + s * r.gvec[2 * nn + n];
        } else {
            const double s = lam * (q[n] - q[4 * nn + n] / r.theta0[n]);
            x = q[nn + n] - s * r.gvec[n];
            y = q[2 * nn + n] - s * r.gvec[nn + n];
            z = q[3 * nn + n] - s * r.gvec[2 * nn + n];
        }
        if (!r.w_zero) {
            const double sc = (lam * lam) / r.theta0[n];
            const double u0 = sc * r.gvec[n], u1 = sc * r.gvec[nn + n], u2 = sc * r.gvec[2 * nn + n];
            const double den = 1.0 + dot3(r.gth0, nn, n, u0, u1, u2);
            if (fabs(den) < 1e-12) atomicOr(a.flags, HEVI_F_AINV);
            const double wv = dot3(r.gth0, nn, n, x, y, z) / den;
            x = x - u0 * wv;
            y = y - u1 * wv;
            z = z - u2 * wv;
        }
        g_project(g, g.bslot[n], x, y, z);
        a.vec[n] = x;
        a.vec[nn + n] = y;
        a.vec[2 * nn + n] = z;
        s0[t] = (x * v0 + y * v1) + z * v2;
    } else if (kind == 2) {
        s0[t] = a.x[n];
    } else {
        s0[t] = (a.vec[n] * v0 + a.vec[nn + n] * v1) + a.vec[2 * nn + n] * v2;
    }
    __syncthreads();
    const int i = t % NQ, j = (t / NQ) % NQ, k = t / (NQ * NQ);
    a.d0[n] = g.Jtv[n] * g_dt<NQ>(s0, sD, i, j, k);
    if (kind == 0) a.d1[n] = g.Jtv[n] * g_dt<NQ>(s1, sD, i, j, k);
}

// ---------------------------------------------------------------------------
// pointwise completions after the DSS of the vertical derivatives
// ---------------------------------------------------------------------------
// L_V(q) (euler.py:331-365) from dP = DSS(Jtv dt P_lin), dV = DSS(Jtv dt (u . vert))
__global__ void kg_lv(const GGeo g, const GRef r, const double* __restrict__ q, const double* __restrict__ dP,
                      const double* __restrict__ dV, double* __restrict__ out) {
    const long long nn = g.nn;
    for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < nn; n += (long long)gridDim.x * blockDim.x) {
        const double v0 = g.vert[n], v1 = g.vert[nn + n], v2 = g.vert[2 * nn + n];
        const double vv = (q[nn + n] * v0 + q[2 * nn + n] * v1) + q[3 * nn + n] * v2;
        const double a0 = vv * v0, a1 = vv * v1, a2 = vv * v2;     // uvert
        const double gP0 = dP[n] * v0, gP1 = dP[n] * v1, gP2 = dP[n] * v2;
        const double q0 = q[n];
        double m0, m1, m2;
        if (r.eqset == 0) {
            out[n] = -(dot3(r.grho0, nn, n, a0, a1, a2) + r.rho0[n] * dV[n]);
            const double rr = r.rho0[n], qr = q0 / rr;
            m0 = -(gP0 / rr + qr * r.gvec[n]);
            m1 = -(gP1 / rr + qr * r.gvec[nn + n]);
            m2 = -(gP2 / rr + qr * r.gvec[2 * nn + n]);
            out[4 * nn + n] = -dot3(r.gth0, nn, n, a0, a1, a2);
        } else {
            out[n] = -dV[n];
            m0 = -(gP0 + q0 * r.gvec[n]);
            m1 = -(gP1 + q0 * r.gvec[nn + n]);
            m2 = -(gP2 + q0 * r.gvec[2 * nn + n]);
            out[4 * nn + n] = -(r.theta0[n] * dV[n] + dot3(r.gth0, nn, n, a0, a1, a2));
        }
        const double mv = (m0 * v0 + m1 * v1) + m2 * v2;
        double x = mv * v0, y = mv * v1, z = mv * v2;
        g_project(g, g.bslot[n], x, y, z);
        out[nn + n] = x;
        out[2 * nn + n] = y;
        out[3 * nn + n] = z;
    }
}

// _up(P) (imexcore.py:245-257) from dP = DSS(Jtv dt P); up -> vec [3][nn]
__device__ __forceinline__ void g_up(const GGeo& g, const GRef& r, long long n, double lam, double P, double dPn,
                                     double& x, double& y, double& z, unsigned* flags) {
    const long long nn = g.nn;
    const double v0 = g.vert[n], v1 = g.vert[nn + n], v2 = g.vert[2 * nn + n];
    const double gP0 = dPn * v0, gP1 = dPn * v1, gP2 = dPn * v2;
    if (r.eqset == 0) {
        const double rr = r.rho0[n], s = P / (r.G0[n] * rr);
        x = lam * (gP0 / rr + s * r.gvec[n]);
        y = lam * (gP1 / rr + s * r.gvec[nn + n]);
        z = lam * (gP2 / rr + s * r.gvec[2 * nn + n]);
    } else {
        const double s = P / (r.F0c[n] * r.theta0[n]);
        x = lam * (gP0 + s * r.gvec[n]);
        y = lam * (gP1 + s * r.gvec[nn + n]);
        z = lam * (gP2 + s * r.gvec[2 * nn + n]);
    }
    if (!r.w_zero) {
        const double sc = (lam * lam) / r.theta0[n];
        const double u0 = sc * r.gvec[n], u1 = sc * r.gvec[nn + n], u2 = sc * r.gvec[2 * nn + n];
        const double den = 1.0 + dot3(r.gth0, nn, n, u0, u1, u2);
        if (fabs(den) < 1e-12) atomicOr(flags, HEVI_F_AINV);
        const double wv = dot3(r.gth0, nn, n, x, y, z) / den;
        x = x - u0 * wv;
        y = y - u1 * wv;
        z = z - u2 * wv;
    }
    g_project(g, g.bslot[n], x, y, z);
}

// lam-scaled Helmholtz flux of a velocity-like field (imexcore._helmholtz_flux, :259-268)
__device__ __forceinline__ double g_helm(const GRef& r, long long n, long long nn, double lam, double x, double y,
                                         double z, double dV) {
    if (r.eqset == 0) return lam * (dot3(r.F0v, nn, n, x, y, z) + (r.rho0[n] * r.G0[n]) * dV);
    return (r.F0c[n] * lam) * (r.theta0[n] * dV + dot3(r.gth0, nn, n, x, y, z));
}

// Schur RHS Pe - flux(ua) (rhs_schur_build), ua in vec
__global__ void kg_schur_rhs(const GGeo g, const GRef r, const double* __restrict__ qe, const double* __restrict__ ua,
                             const double* __restrict__ dV, double lam, double* __restrict__ rhs) {
    const long long nn = g.nn;
    for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < nn; n += (long long)gridDim.x * blockDim.x) {
        const double Pe = r.eqset == 0 ? r.G0[n] * qe[n] + r.H0[n] * qe[4 * nn + n] : r.F0c[n] * qe[4 * nn + n];
        rhs[n] = Pe - g_helm(r, n, nn, lam, ua[n], ua[nn + n], ua[2 * nn + n], dV[n]);
    }
}

// up(P) into vec (the probe's first half) and its vertical component plane
__global__ void kg_up(const GGeo g, const GRef r, const double* __restrict__ P, const double* __restrict__ dP,
                      double lam, double* __restrict__ up, unsigned* flags) {
    const long long nn = g.nn;
    for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < nn; n += (long long)gridDim.x * blockDim.x) {
        double x, y, z;
        g_up(g, r, n, lam, P[n], dP[n], x, y, z, flags);
        up[n] = x;
        up[nn + n] = y;
        up[2 * nn + n] = z;
    }
}

// lhs_schur(P) = P - flux(up(P)) (imexcore.py:270-271)
__global__ void kg_lhs(const GGeo g, const GRef r, const double* __restrict__ P, const double* __restrict__ up,
                       const double* __restrict__ dV, double lam, double* __restrict__ out) {
    const long long nn = g.nn;
    for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < nn; n += (long long)gridDim.x * blockDim.x)
        out[n] = P[n] - g_helm(r, n, nn, lam, up[n], up[nn + n], up[2 * nn + n], dV[n]);
}

// extract_from_pressure (imexcore.py:273-298), dim = 1d
__global__ void kg_extract(const GGeo g, const GRef r, const double* __restrict__ P, const double* __restrict__ dP,
                           const double* __restrict__ ua, const double* __restrict__ qe, double lam,
                           double* __restrict__ q, unsigned* flags) {
    const long long nn = g.nn;
    for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < nn; n += (long long)gridDim.x * blockDim.x) {
        double x, y, z;
        const double Pn = P[n];
        g_up(g, r, n, lam, Pn, dP[n], x, y, z, flags);
        const double w0 = ua[n] - x, w1 = ua[nn + n] - y, w2 = ua[2 * nn + n] - z;
        const double v0 = g.vert[n], v1 = g.vert[nn + n], v2 = g.vert[2 * nn + n];
        const double uv = (w0 * v0 + w1 * v1) + w2 * v2;
        const double a0 = uv * v0, a1 = uv * v1, a2 = uv * v2;
        double q0, q4;
        if (r.eqset == 0) {
            q4 = qe[4 * nn + n] - lam * dot3(r.gth0, nn, n, a0, a1, a2);
            q0 = (Pn - r.H0[n] * q4) / r.G0[n];
        } else {
            const double G0 = r.theta0[n];
            q4 = Pn / r.F0c[n];
            q0 = ((Pn / (r.F0c[n] * G0) + lam / G0 * dot3(r.gth0, nn, n, a0, a1, a2)) - qe[4 * nn + n] / G0) + qe[n];
        }
        q[n] = q0;
        q[nn + n] = w0;
        q[2 * nn + n] = w1;
        q[3 * nn + n] = w2;
        q[4 * nn + n] = q4;
    }
}

// ---------------------------------------------------------------------------
// unique (column, level) space (columnsolve.unique_space, :27-61)
// ---------------------------------------------------------------------------
__global__ void kg_gather(const double* __restrict__ f, const int* __restrict__ rep, double* __restrict__ col, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        col[i] = f[rep[i]];
}

__global__ void kg_scatter(const double* __restrict__ col, const int* __restrict__ uid, double* __restrict__ f, long long nn) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nn; i += (long long)gridDim.x * blockDim.x)
        f[i] = col[uid[i]];
}

// probe vector: 1 at level `lev` of every column (or of column `only` when >= 0)
__global__ void kg_probe_vec(const int* __restrict__ uid, int n_lev, int lev, int only, double* __restrict__ P, long long nn) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nn; i += (long long)gridDim.x * blockDim.x) {
        const int u = uid[i];
        P[i] = (u % n_lev == lev && (only < 0 || u / n_lev == only)) ? 1.0 : 0.0;
    }
}

// column `lev` of every column's matrix: A[c][row][lev] = out[rep[c*M + row]]
__global__ void kg_probe_store(const double* __restrict__ out, const int* __restrict__ rep, int n_col, int M, int lev,
                               double* __restrict__ A) {
    const long long n = (long long)n_col * M;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        A[i * M + lev] = out[rep[i]];
}

// max |x| as ordered bits (non-negative doubles order like their bit patterns)
__global__ void kg_absmax_bits(const double* __restrict__ x, long long n, long long skip0, long long skip1,
                               unsigned long long* out) {
    unsigned long long m = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        if (i >= skip0 && i < skip1) continue;
        const unsigned long long b = (unsigned long long)__double_as_longlong(fabs(x[i]));
        m = b > m ? b : m;
    }
    atomicMax(out, m);
}

// bandwidth of the probed pattern (columnsolve.py:103-107): max |row - col| + 1
// over entries above 1e-14 of the largest magnitude
__global__ void kg_bandwidth(const double* __restrict__ A, int n_col, int M, const unsigned long long* scale_bits,
                             int* nb) {
    const double thr = 1e-14 * __longlong_as_double((long long)*scale_bits);
    const long long n = (long long)n_col * M * M;
    int b = 1;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int cc = (int)(i % M), rr = (int)((i / M) % M);
        if (fabs(A[i]) > thr) b = max(b, abs(rr - cc) + 1);
    }
    atomicMax(nb, b);
}

// ---------------------------------------------------------------------------
// stage combinations of the steppers
// ---------------------------------------------------------------------------
// ARK predictor (imexcore.py:400-403): out = q + sum_j dt (a_j (R_j - L_j) + at_j L_j), j < nj
__global__ void kg_pred(const double* __restrict__ q, const double* __restrict__ R0, const double* __restrict__ L0,
                        const double* __restrict__ R1, const double* __restrict__ L1, int nj, double dt, double a0,
                        double at0, double a1, double at1, double* __restrict__ out, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double p = q[i] + dt * (a0 * (R0[i] - L0[i]) + at0 * L0[i]);
        if (nj > 1) p = p + dt * (a1 * (R1[i] - L1[i]) + at1 * L1[i]);
        out[i] = p;
    }
}

// ARK final combination (imexcore.py:409-411): out = q + sum_i (dt b_i) R_i; non-finite flag
__global__ void kg_final(const double* q, const double* __restrict__ R0, const double* __restrict__ R1,
                         const double* __restrict__ R2, double c0, double c1, double c2, double* out, long long n,
                         unsigned* flags) {
    bool bad = false;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double v = ((q[i] + c0 * R0[i]) + c1 * R1[i]) + c2 * R2[i];
        out[i] = v;
        bad = bad || !isfinite(v);
    }
    if (bad) atomicOr(flags, HEVI_F_NONFINITE_OUT);
}

// RK35 stage accumulation (imexcore.py:111-126): acc = sum_k c_k x_k in order
struct GTerms {
    const double* x[4];
    double c[4];
    int n;
};
__global__ void kg_terms(const GTerms T, double* out, long long n, int check, unsigned* flags) {
    bool bad = false;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double a = 0.0;
        for (int k = 0; k < T.n; ++k) a = a + T.c[k] * T.x[k][i];
        out[i] = a;
        bad = bad || !isfinite(a);
    }
    if (check && bad) atomicOr(flags, HEVI_F_NONFINITE_OUT);
}

// DSS-projected gradient / divergence before DSS (Discretization.gradc / divc,
// euler.py:281-290): grad -> 3 planes, div -> 1 plane
template <int NQ>
__global__ void __launch_bounds__(NQ * NQ * NQ) kg_graddiv(const GGeo g, const double* __restrict__ in, int div,
                                                           double* __restrict__ out) {
    constexpr int NP = NQ * NQ * NQ;
    __shared__ double s[3][NP];
    __shared__ double sD[NQ * NQ];
    const int t = threadIdx.x;
    const long long n = (long long)blockIdx.x * NP + t;
    const long long nn = g.nn;
    for (int i = t; i < NQ * NQ; i += NP) sD[i] = g.D[i];
    const int nf = div ? 3 : 1;
    for (int f = 0; f < nf; ++f) s[f][t] = in[f * nn + n];
    __syncthreads();
    const int i = t % NQ, j = (t / NQ) % NQ, k = t / (NQ * NQ);
    double fr, fs, ft;
    if (!div) {
        g_d3<NQ>(s[0], sD, i, j, k, fr, fs, ft);
        for (int c = 0; c < 3; ++c) out[c * nn + n] = g_gc(g, n, c, fr, fs, ft);
    } else {
        double d = 0.0;
        for (int m = 0; m < 3; ++m) {
            g_d3<NQ>(s[m], sD, i, j, k, fr, fs, ft);
            const long long o = m * nn + n;
            d = d + fr * g.ar[o];
            d = d + fs * g.as[o];
            d = d + ft * g.at[o];
        }
        out[n] = d;
    }
}

// times the vertical unit vector: out_c = d * vert_c (grad_vc)
__global__ void kg_times_vert(const GGeo g, const double* __restrict__ d, double* __restrict__ out) {
    const long long nn = g.nn;
    for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < nn; n += (long long)gridDim.x * blockDim.x) {
        const double v = d[n];
        out[n] = v * g.vert[n];
        out[nn + n] = v * g.vert[nn + n];
        out[2 * nn + n] = v * g.vert[2 * nn + n];
    }
}

// ---------------------------------------------------------------------------
// 3D-IMEX pieces on the general mesh (ImplicitProblem dim = "3d",
// imexcore.py:200-298 with gradc / divc): pointwise parts; the DSS-projected
// gradient / divergence come from kg_graddiv + kg_dss
// ---------------------------------------------------------------------------
// A^-1 v (imexcore._ainv, :200-216) and the no-flux projection of the node
__device__ __forceinline__ void g_ainv_proj(const GGeo& g, const GRef& r, long long n, double lam, double& x,
                                            double& y, double& z, unsigned* flags) {
    const long long nn = g.nn;
    if (!r.w_zero) {
        const double sc = (lam * lam) / r.theta0[n];
        const double u0 = sc * r.gvec[n], u1 = sc * r.gvec[nn + n], u2 = sc * r.gvec[2 * nn + n];
        const double den = 1.0 + dot3(r.gth0, nn, n, u0, u1, u2);
        if (fabs(den) < 1e-12) atomicOr(flags, HEVI_F_AINV);
        const double wv = dot3(r.gth0, nn, n, x, y, z) / den;
        x = x - u0 * wv;
        y = y - u1 * wv;
        z = z - u2 * wv;
    }
    g_project(g, g.bslot[n], x, y, z);
}

// rhs_schur_build's ua and Pe (imexcore.py:229-243): ua -> [3][nn], Pe -> [nn]
__global__ void kg_schur_ua(const GGeo g, const GRef r, const double* __restrict__ qe, double lam,
                            double* __restrict__ ua, double* __restrict__ Pe, unsigned* flags) {
    const long long nn = g.nn;
    for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < nn; n += (long long)gridDim.x * blockDim.x) {
        double x, y, z;
        if (r.eqset == 0) {
            const double s = ((lam * r.H0[n]) / (r.G0[n] * r.rho0[n])) * qe[4 * nn + n];
            x = qe[nn + n] + s * r.gvec[n];
            y = qe[2 * nn + n] + s * r.gvec[nn + n];
            z = qe[3 * nn + n] + s * r.gvec[2 * nn + n];
            Pe[n] = r.G0[n] * qe[n] + r.H0[n] * qe[4 * nn + n];
        } else {
            const double s = lam * (qe[n] - qe[4 * nn + n] / r.theta0[n]);
            x = qe[nn + n] - s * r.gvec[n];
            y = qe[2 * nn + n] - s * r.gvec[nn + n];
            z = qe[3 * nn + n] - s * r.gvec[2 * nn + n];
            Pe[n] = r.F0c[n] * qe[4 * nn + n];
        }
        g_ainv_proj(g, r, n, lam, x, y, z, flags);
        ua[n] = x;
        ua[nn + n] = y;
        ua[2 * nn + n] = z;
    }
}

// _up(P) from the DSS-projected gradient gP [3][nn] (imexcore.py:245-257)
__global__ void kg_up3(const GGeo g, const GRef r, const double* __restrict__ P, const double* __restrict__ gP,
                       double lam, double* __restrict__ up, unsigned* flags) {
    const long long nn = g.nn;
    for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < nn; n += (long long)gridDim.x * blockDim.x) {
        double x, y, z;
        if (r.eqset == 0) {
            const double rr = r.rho0[n], s = P[n] / (r.G0[n] * rr);
            x = lam * (gP[n] / rr + s * r.gvec[n]);
            y = lam * (gP[nn + n] / rr + s * r.gvec[nn + n]);
            z = lam * (gP[2 * nn + n] / rr + s * r.gvec[2 * nn + n]);
        } else {
            const double s = P[n] / (r.F0c[n] * r.theta0[n]);
            x = lam * (gP[n] + s * r.gvec[n]);
            y = lam * (gP[nn + n] + s * r.gvec[nn + n]);
            z = lam * (gP[2 * nn + n] + s * r.gvec[2 * nn + n]);
        }
        g_ainv_proj(g, r, n, lam, x, y, z, flags);
        up[n] = x;
        up[nn + n] = y;
        up[2 * nn + n] = z;
    }
}

// extract_from_pressure (imexcore.py:273-298); vo: 1d (advection by the
// vertical part of the velocity) or 3d (the whole velocity)
__global__ void kg_extract3(const GGeo g, const GRef r, const double* __restrict__ P, const double* __restrict__ ua,
                            const double* __restrict__ up, const double* __restrict__ qe, double lam, int vo,
                            double* __restrict__ q) {
    const long long nn = g.nn;
    for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < nn; n += (long long)gridDim.x * blockDim.x) {
        const double w0 = ua[n] - up[n], w1 = ua[nn + n] - up[nn + n], w2 = ua[2 * nn + n] - up[2 * nn + n];
        double a0 = w0, a1 = w1, a2 = w2;
        if (vo) {
            const double v0 = g.vert[n], v1 = g.vert[nn + n], v2 = g.vert[2 * nn + n];
            const double uv = (w0 * v0 + w1 * v1) + w2 * v2;
            a0 = uv * v0;
            a1 = uv * v1;
            a2 = uv * v2;
        }
        const double Pn = P[n];
        double q0, q4;
        if (r.eqset == 0) {
            q4 = qe[4 * nn + n] - lam * dot3(r.gth0, nn, n, a0, a1, a2);
            q0 = (Pn - r.H0[n] * q4) / r.G0[n];
        } else {
            const double G0 = r.theta0[n];
            q4 = Pn / r.F0c[n];
            q0 = ((Pn / (r.F0c[n] * G0) + lam / G0 * dot3(r.gth0, nn, n, a0, a1, a2)) - qe[4 * nn + n] / G0) + qe[n];
        }
        q[n] = q0;
        q[nn + n] = w0;
        q[2 * nn + n] = w1;
        q[3 * nn + n] = w2;
        q[4 * nn + n] = q4;
    }
}

// the full 3D linear operator (euler.linear_operator, dim 3d, euler.py:313-365)
// from gP = gradc(P_lin) [3][nn] and dV = divc(velocity) [nn]
__global__ void kg_lin3(const GGeo g, const GRef r, const double* __restrict__ q, const double* __restrict__ gP,
                        const double* __restrict__ dV, double* __restrict__ out) {
    const long long nn = g.nn;
    for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < nn; n += (long long)gridDim.x * blockDim.x) {
        const double u0 = q[nn + n], u1 = q[2 * nn + n], u2 = q[3 * nn + n], q0 = q[n];
        double m0, m1, m2;
        if (r.eqset == 0) {
            out[n] = -(dot3(r.grho0, nn, n, u0, u1, u2) + r.rho0[n] * dV[n]);
            const double rr = r.rho0[n], qr = q0 / rr;
            m0 = -(gP[n] / rr + qr * r.gvec[n]);
            m1 = -(gP[nn + n] / rr + qr * r.gvec[nn + n]);
            m2 = -(gP[2 * nn + n] / rr + qr * r.gvec[2 * nn + n]);
            out[4 * nn + n] = -dot3(r.gth0, nn, n, u0, u1, u2);
        } else {
            out[n] = -dV[n];
            m0 = -(gP[n] + q0 * r.gvec[n]);
            m1 = -(gP[nn + n] + q0 * r.gvec[nn + n]);
            m2 = -(gP[2 * nn + n] + q0 * r.gvec[2 * nn + n]);
            out[4 * nn + n] = -(r.theta0[n] * dV[n] + dot3(r.gth0, nn, n, u0, u1, u2));
        }
        g_project(g, g.bslot[n], m0, m1, m2);
        out[nn + n] = m0;
        out[2 * nn + n] = m1;
        out[3 * nn + n] = m2;
    }
}

// linearised pressure of the state (euler.py:188-194) -> [nn]
__global__ void kg_plin(const GGeo g, const GRef r, const double* __restrict__ q, double* __restrict__ P) {
    const long long nn = g.nn;
    for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < nn; n += (long long)gridDim.x * blockDim.x)
        P[n] = r.eqset == 0 ? r.G0[n] * q[n] + r.H0[n] * q[4 * nn + n] : r.F0c[n] * q[4 * nn + n];
}

// plain dot product over n doubles in a fixed order (the reference's np.dot
// over E-vectors, krylov.py:46-55): per-block partial sums, then one thread
__global__ void kg_dot(const double* __restrict__ x, const double* __restrict__ y, long long n, double* part) {
    __shared__ double sm[KV_T];
    double s = 0.0;
    for (long long i = (long long)blockIdx.x * KV_T + threadIdx.x; i < n; i += (long long)KV_BLOCKS * KV_T)
        s = fma(x[i], y[i], s);
    sm[threadIdx.x] = s;
    __syncthreads();
    for (int t = KV_T / 2; t > 0; t >>= 1) {
        if (threadIdx.x < t) sm[threadIdx.x] += sm[threadIdx.x + t];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sm[0];
}
