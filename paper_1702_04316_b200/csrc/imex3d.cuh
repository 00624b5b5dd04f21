// imex3d.cuh -- operators of the 3D-IMEX Schur solve and the full linear
// operator (included by hevi.cu inside its anonymous
// namespace).
//
// imexcore.ImplicitProblem with dim="3d" (imexcore.py:200-271) reduces the
// implicit problem to the pressure equation
//     lhs_schur(P) = P - helmholtz_flux(up(P))
// with full DSS-projected gradients / divergences (euler.py:281-290), solved
// matrix-free by Krylov iterations (krylov.py).  On the unique lattice every
// DSS-projected derivative is the folded derivative of the explicit kernels
// (DESIGN.md "folded DSS"), so each operator below is one pass, one thread
// per lattice point, reading its element lines through L1/L2:
//   k3_linear   euler.linear_operator, vertical_only=False (euler.py:313-365)
//   k3_up       ImplicitProblem._up (imexcore.py:245-257)
//   k3_flux     a*P - _helmholtz_flux(vel) (imexcore.py:259-268): lhs_schur
//               (a = 1, vel = up) and the Schur rhs (P = Pe, vel = ua)
//   k3_ua       the ua / Pe part of rhs_schur_build (imexcore.py:229-243)
//   k3_extract  extract_from_pressure, dim="3d" (imexcore.py:273-298)
// plus the Krylov vector kernels: the multiplicity-weighted dot product
// (the reference's Krylov vectors are E-vectors, where every lattice point
// appears once per element copy; a continuous field's E-vector dot product is
// sum_g m_g a_g b_g with m_g = m_x m_y m_z copies) and y = a x + b y.
#pragma once

struct I3Args {
    Geo g;
    Lev lv;
    Phys ph;
    const double *cx, *cy, *cz, *Dx, *Dy, *Dz;
    int N, Ny, eqset, ainv_identity;
    int vert_only;   // dim = "1d": grad_vc / div_vc (euler.py:292-300) instead of gradc / divc
    double lam;
};

// folded d/d(axis) at lattice index gi of the axis: own element row first,
// then the lower element's row N on an element face (same order as the
// explicit kernels).  val(j) = field value at axis index j.
template <class F>
__device__ __forceinline__ double fold_d(F&& val, int gi, int N, int ne, const double* __restrict__ D) {
    int row, s0;
    bool face;
    if (gi == ne * N) {
        row = N;
        s0 = gi - N;
        face = false;
    } else {
        row = gi % N;
        s0 = gi - row;
        face = (row == 0) && (gi > 0);
    }
    double d = 0.0;
    for (int m = 0; m <= N; ++m) d = fma(__ldg(D + row * (N + 1) + m), val(s0 + m), d);
    if (face) {
        double e = 0.0;
        for (int m = 0; m <= N; ++m) e = fma(__ldg(D + N * (N + 1) + m), val(gi - N + m), e);
        d += e;
    }
    return d;
}

struct P3 {
    int gx, gy, gz;
    long long o;
    bool ok;
};

__device__ __forceinline__ P3 point3(const Geo& g, long long i) {
    P3 p;
    const int x = (int)(i % g.lX);
    const long long t = i / g.lX;
    const int y = (int)(t % g.lY);
    p.gz = (int)(t / g.lY);
    p.gx = x + g.x0;
    p.gy = y + g.y0;
    p.o = ((long long)p.gz * g.lY + y) * g.px + x;
    p.ok = p.gz < g.Z;
    return p;
}

// gradient of a per-point scalar s(o, gz) at point p (cx, cy, cz applied)
template <class S>
__device__ __forceinline__ void grad3(const I3Args& a, const P3& p, S&& s, double& gx, double& gy,
                                      double& gz) {
    const Geo& g = a.g;
    const long long sx = 1, sy = g.px, sz = (long long)g.lY * g.px;
    if (a.vert_only) {
        gx = 0.0;
        gy = 0.0;
    } else {
        gx = __ldg(a.cx + p.gx) *
             fold_d([&](int j) { return s(p.o + (j - p.gx) * sx, p.gz); }, p.gx, a.N, g.nex, a.Dx);
        gy = __ldg(a.cy + p.gy) *
             fold_d([&](int j) { return s(p.o + (j - p.gy) * sy, p.gz); }, p.gy, a.Ny, g.ney, a.Dy);
    }
    gz = __ldg(a.cz + p.gz) *
         fold_d([&](int j) { return s(p.o + (j - p.gz) * sz, j); }, p.gz, a.N, g.nez, a.Dz);
}

// DSS-projected divergence of the 3-field vector v (field stride fs)
__device__ __forceinline__ double div3(const I3Args& a, const P3& p, const double* __restrict__ v) {
    const Geo& g = a.g;
    const long long fs = g.fs, sy = g.px, sz = (long long)g.lY * g.px;
    if (a.vert_only)
        return __ldg(a.cz + p.gz) *
            fold_d([&](int j) { return __ldg(v + 2 * fs + p.o + (j - p.gz) * sz); }, p.gz, a.N, g.nez, a.Dz);
    const double dx = __ldg(a.cx + p.gx) *
        fold_d([&](int j) { return __ldg(v + p.o + (j - p.gx)); }, p.gx, a.N, g.nex, a.Dx);
    const double dy = __ldg(a.cy + p.gy) *
        fold_d([&](int j) { return __ldg(v + fs + p.o + (j - p.gy) * sy); }, p.gy, a.Ny, g.ney, a.Dy);
    const double dz = __ldg(a.cz + p.gz) *
        fold_d([&](int j) { return __ldg(v + 2 * fs + p.o + (j - p.gz) * sz); }, p.gz, a.N, g.nez, a.Dz);
    return (dx + dy) + dz;
}

// rank-one inverse of A = I + lam^2 u w^T (imexcore.py:200-217): u, w vertical
__device__ __forceinline__ double ainv_z(const I3Args& a, int k, double vz) {
    if (a.ainv_identity) return vz;
    const double th0 = a.lv.theta0[k], dth0 = a.lv.dth0[k];
    const double u = (a.lam * a.lam / th0) * a.ph.g;
    const double den = 1.0 + dth0 * u;
    return vz - u * ((dth0 * vz) / den);
}

__device__ __forceinline__ void boundary3(const Geo& g, const P3& p, bool& bx, bool& by, bool& bz) {
    bx = (p.gx == 0) || (p.gx == g.X - 1);
    by = g.slab || (p.gy == 0) || (p.gy == g.Y - 1);
    bz = (p.gz == 0) || (p.gz == g.Z - 1);
}

// linearised pressure of q at (offset, level)
__device__ __forceinline__ double plin(const I3Args& a, const double* __restrict__ q, long long o, int k) {
    if (a.eqset == 1) return a.lv.F0c[k] * __ldg(q + o + 4 * a.g.fs);
    return a.lv.G0[k] * __ldg(q + o) + a.lv.H0[k] * __ldg(q + o + 4 * a.g.fs);
}

__global__ void k3_linear(const I3Args a, const double* __restrict__ q, double* __restrict__ out) {
    const Geo& g = a.g;
    const long long n = (long long)g.Z * g.lY * g.lX;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const P3 p = point3(g, i);
    const int k = p.gz;
    const long long fs = g.fs;
    double gPx, gPy, gPz;
    grad3(a, p, [&](long long o, int kk) { return plin(a, q, o, kk); }, gPx, gPy, gPz);
    const double divU = div3(a, p, q + fs);
    const double r = __ldg(q + p.o), u = __ldg(q + p.o + fs), v = __ldg(q + p.o + 2 * fs),
                 w = __ldg(q + p.o + 3 * fs);
    (void)u;
    (void)v;
    const double rho0 = a.lv.rho0[k], gr = a.ph.g;
    double o0, mx, my, mz, o4;
    if (a.eqset == 1) {   // euler.py:350-354
        o0 = -divU;
        mx = -gPx;
        my = -gPy;
        mz = -(gPz + r * gr);
        o4 = -(a.lv.theta0[k] * divU + w * a.lv.dth0[k]);
    } else {              // euler.py:346-349
        o0 = -(w * a.lv.drho0[k] + rho0 * divU);
        mx = -(gPx / rho0);
        my = -(gPy / rho0);
        mz = -(gPz / rho0 + (r / rho0) * gr);
        o4 = -(w * a.lv.dth0[k]);
    }
    bool bx, by, bz;
    boundary3(g, p, bx, by, bz);
    out[p.o] = o0;
    out[p.o + fs] = bx ? 0.0 : mx;
    out[p.o + 2 * fs] = by ? 0.0 : my;
    out[p.o + 3 * fs] = bz ? 0.0 : mz;
    out[p.o + 4 * fs] = o4;
}

// up = A^-1 lam (grad P / rho0 + P/(G0 rho0) g z)  [set2c: grad P + P/(F0 G0) g z]
__global__ void k3_up(const I3Args a, const double* __restrict__ P, double* __restrict__ up) {
    const Geo& g = a.g;
    const long long n = (long long)g.Z * g.lY * g.lX;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const P3 p = point3(g, i);
    const int k = p.gz;
    double gx, gy, gz;
    grad3(a, p, [&](long long o, int) { return __ldg(P + o); }, gx, gy, gz);
    const double Pk = __ldg(P + p.o), lam = a.lam, gr = a.ph.g;
    double vx, vy, vz;
    if (a.eqset == 1) {
        const double th0 = a.lv.theta0[k];
        vx = lam * gx;
        vy = lam * gy;
        vz = lam * (gz + (Pk / (a.lv.F0c[k] * th0)) * gr);
    } else {
        const double rho0 = a.lv.rho0[k];
        vx = lam * (gx / rho0);
        vy = lam * (gy / rho0);
        vz = lam * (gz / rho0 + (Pk / (a.lv.G0[k] * rho0)) * gr);
    }
    vz = ainv_z(a, k, vz);
    bool bx, by, bz;
    boundary3(g, p, bx, by, bz);
    const long long fs = g.fs;
    up[p.o] = bx ? 0.0 : vx;
    up[p.o + fs] = by ? 0.0 : vy;
    up[p.o + 2 * fs] = bz ? 0.0 : vz;
}

// out = P - helmholtz_flux(vel)
__global__ void k3_flux(const I3Args a, const double* __restrict__ P, const double* __restrict__ vel,
                        double* __restrict__ out) {
    const Geo& g = a.g;
    const long long n = (long long)g.Z * g.lY * g.lX;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const P3 p = point3(g, i);
    const int k = p.gz;
    const double dv = div3(a, p, vel);
    const double vz = __ldg(vel + p.o + 2 * g.fs);
    double flux;
    if (a.eqset == 1)   // imexcore.py:267-268
        flux = a.lv.F0c[k] * a.lam * (a.lv.theta0[k] * dv + a.lv.dth0[k] * vz);
    else                // imexcore.py:264-265
        flux = a.lam * (a.lv.F0z[k] * vz + a.lv.rho0G0[k] * dv);
    out[p.o] = __ldg(P + p.o) - flux;
}

// ua (3 fields) and Pe of rhs_schur_build
__global__ void k3_ua(const I3Args a, const double* __restrict__ qe, double* __restrict__ ua,
                      double* __restrict__ Pe) {
    const Geo& g = a.g;
    const long long n = (long long)g.Z * g.lY * g.lX;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const P3 p = point3(g, i);
    const int k = p.gz;
    const long long fs = g.fs;
    const double re = qe[p.o], ue = qe[p.o + fs], ve = qe[p.o + 2 * fs], we = qe[p.o + 3 * fs],
                 te = qe[p.o + 4 * fs];
    const double lam = a.lam, gr = a.ph.g;
    double vz;
    if (a.eqset == 1) {
        vz = we - (lam * (re - te / a.lv.theta0[k])) * gr;
        Pe[p.o] = a.lv.F0c[k] * te;
    } else {
        const double coef = lam * a.lv.H0[k] / (a.lv.G0[k] * a.lv.rho0[k]);
        vz = we + (coef * te) * gr;
        Pe[p.o] = a.lv.G0[k] * re + a.lv.H0[k] * te;
    }
    vz = ainv_z(a, k, vz);
    bool bx, by, bz;
    boundary3(g, p, bx, by, bz);
    ua[p.o] = bx ? 0.0 : ue;
    ua[p.o + fs] = by ? 0.0 : ve;
    ua[p.o + 2 * fs] = bz ? 0.0 : vz;
}

// q from P, ua, up and q_e (imexcore.py:273-298, dim = "3d")
__global__ void k3_extract(const I3Args a, const double* __restrict__ P, const double* __restrict__ ua,
                           const double* __restrict__ up, const double* __restrict__ qe,
                           double* __restrict__ q) {
    const Geo& g = a.g;
    const long long n = (long long)g.Z * g.lY * g.lX;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const P3 p = point3(g, i);
    const int k = p.gz;
    const long long fs = g.fs;
    const double vx = ua[p.o] - up[p.o], vy = ua[p.o + fs] - up[p.o + fs],
                 vz = ua[p.o + 2 * fs] - up[p.o + 2 * fs];
    const double Pk = P[p.o], lam = a.lam;
    q[p.o + fs] = vx;
    q[p.o + 2 * fs] = vy;
    q[p.o + 3 * fs] = vz;
    const double dth0 = a.lv.dth0[k];
    if (a.eqset == 1) {
        const double F0 = a.lv.F0c[k], G0 = a.lv.theta0[k];
        q[p.o + 4 * fs] = Pk / F0;
        q[p.o] = ((Pk / (F0 * G0) + lam / G0 * (vz * dth0)) - qe[p.o + 4 * fs] / G0) + qe[p.o];
    } else {
        const double th = qe[p.o + 4 * fs] - lam * (vz * dth0);
        q[p.o + 4 * fs] = th;
        q[p.o] = (Pk - a.lv.H0[k] * th) / a.lv.G0[k];
    }
}

// DSS-projected gradient of a scalar (Discretization.gradc / grad_vc,
// euler.py:281-295): out = (d/dx, d/dy, d/dz) f, three fields; with
// vert_only the x, y components are zero (grad_vc multiplies the vertical
// derivative by vert = z on a box)
__global__ void k3_grad(const I3Args a, const double* __restrict__ f, double* __restrict__ out) {
    const Geo& g = a.g;
    const long long n = (long long)g.Z * g.lY * g.lX;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const P3 p = point3(g, i);
    double gx, gy, gz;
    grad3(a, p, [&](long long o, int) { return __ldg(f + o); }, gx, gy, gz);
    out[p.o] = gx;
    out[p.o + g.fs] = gy;
    out[p.o + 2 * g.fs] = gz;
}

// DSS-projected divergence of a 3-field vector (Discretization.divc /
// div_vc, euler.py:287-300)
__global__ void k3_div(const I3Args a, const double* __restrict__ vec, double* __restrict__ out) {
    const Geo& g = a.g;
    const long long n = (long long)g.Z * g.lY * g.lX;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const P3 p = point3(g, i);
    out[p.o] = div3(a, p, vec);
}

// ---- Krylov vector kernels -------------------------------------------------
constexpr int KV_BLOCKS = 296, KV_T = 256;

__device__ __forceinline__ double mult_axis(int gi, int N, int ne) {
    return (gi > 0 && gi < ne * N && gi % N == 0) ? 2.0 : 1.0;
}

__global__ void k3_wdot(Geo g, int N, int Ny, int nf, const double* __restrict__ x,
                        const double* __restrict__ y, double* part) {
    __shared__ double sm[KV_T];
    const long long n = (long long)g.Z * g.lY * g.lX;
    double s = 0.0;
    for (long long i = (long long)blockIdx.x * KV_T + threadIdx.x; i < n; i += (long long)KV_BLOCKS * KV_T) {
        const P3 p = point3(g, i);
        const double m = mult_axis(p.gx, N, g.nex) * mult_axis(p.gy, Ny, g.ney) * mult_axis(p.gz, N, g.nez);
        for (int f = 0; f < nf; ++f) s = fma(m * x[p.o + f * g.fs], y[p.o + f * g.fs], s);
    }
    sm[threadIdx.x] = s;
    __syncthreads();
    for (int t = KV_T / 2; t > 0; t >>= 1) {
        if (threadIdx.x < t) sm[threadIdx.x] += sm[threadIdx.x + t];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sm[0];
}

__global__ void k3_sum(const double* part, int n, double* out) {
    if (threadIdx.x != 0) return;
    double s = 0.0;
    for (int b = 0; b < n; ++b) s += part[b];
    *out = s;
}

// y = alpha x + beta y over n contiguous doubles
__global__ void k3_axpby(long long n, double alpha, const double* __restrict__ x, double beta,
                         double* __restrict__ y) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        y[i] = (beta == 0.0) ? alpha * x[i] : fma(alpha, x[i], beta * y[i]);
}
