// general_api.cuh -- C ABI of the general-mesh path (include/hevi.h), inside
// hevi.cu's extern "C" block.

int hevi_gplan_create(hevi_gplan** out, const hevi_gmesh_desc* m, const hevi_gref_desc* rd) {
    if (!out || !m || !rd) return fail("null argument");
    *out = nullptr;
    if (m->N < 1 || m->N > 8 || m->nel < 1) return fail("general mesh: order must be 1..8");
    if (rd->eqset != 0 && rd->eqset != 1) return fail("unknown equation set");
    const int nq = m->N + 1, NP = nq * nq * nq;
    const long long nn = (long long)m->nel * NP;
    if (nn > 0x7fffffffLL) return fail("general mesh too large for 32-bit node indices");
    hevi_gplan* gp = new hevi_gplan();
    gp->nn = nn;
    gp->n_groups = m->n_groups;
    gp->n_proj = m->n_proj;
    gp->n_col = m->n_col;
    gp->n_lev = m->n_lev;
    // double arrays: D | ar as at vert (12 nn) | Jtv w | wsum | proj | rho0 theta0 P0f |
    // grho0 gth0 gvec (9 nn) | G0 H0 | F0v (3 nn) | Th0 F0c | Pb c0 irt0
    const size_t nd = (size_t)nq * nq + 12 * nn + 2 * nn + m->n_groups + 9 * (size_t)m->n_proj + 3 * nn +
                      9 * nn + 2 * nn + 3 * nn + 2 * nn + 3 * nn;
    std::vector<double> h(nd, 0.0);
    size_t o = 0;
    auto put = [&](const double* src, size_t n) {
        double* dst = h.data() + o;
        if (src) memcpy(dst, src, sizeof(double) * n);
        o += n;
        return dst;
    };
    const double* hD = put(m->D, (size_t)nq * nq);
    put(m->ar, 3 * nn);
    put(m->as, 3 * nn);
    put(m->at, 3 * nn);
    put(m->vert, 3 * nn);
    put(m->Jtv, nn);
    put(m->w, nn);
    put(m->grp_wsum, m->n_groups);
    put(m->proj, 9 * (size_t)m->n_proj);
    put(rd->rho0, nn);
    put(rd->theta0, nn);
    put(rd->P0f, nn);
    put(rd->grad_rho0, 3 * nn);
    const double* hgth = put(rd->grad_theta0, 3 * nn);
    put(rd->gvec, 3 * nn);
    put(rd->G0, nn);
    put(rd->H0, nn);
    put(rd->F0vec, 3 * nn);
    put(rd->Theta0, nn);
    put(rd->F0c, nn);
    put(rd->Pb, nn);
    double* hc0 = put(nullptr, nn);
    double* hirt = put(nullptr, nn);
    const size_t base_bg = (size_t)nq * nq + 14 * nn + m->n_groups + 9 * (size_t)m->n_proj;
    for (long long n = 0; n < nn; ++n) {
        hc0[n] = rd->Pb[n] - rd->P0f[n];
        hirt[n] = 1.0 / (rd->rho0[n] * rd->theta0[n]);
    }
    (void)hD;
    int wz = 1;
    for (long long n = 0; n < 3 * nn && wz; ++n) wz = hgth[n] == 0.0;
    // integer arrays: gptr | gidx | gslot | uid | rep | bslot
    const long long nu = (long long)m->n_col * m->n_lev;
    std::vector<int> hi((size_t)(m->n_groups + 1) + nn + m->n_groups + nn + nu + nn);
    int* ip = hi.data();
    memcpy(ip, m->grp_ptr, sizeof(int) * (m->n_groups + 1));
    memcpy(ip + m->n_groups + 1, m->grp_idx, sizeof(int) * nn);
    int* hslot = ip + m->n_groups + 1 + nn;
    for (int gi = 0; gi < m->n_groups; ++gi) hslot[gi] = m->grp_slot ? m->grp_slot[gi] : -1;
    memcpy(hslot + m->n_groups, m->uid, sizeof(int) * nn);
    memcpy(hslot + m->n_groups + nn, m->rep, sizeof(int) * nu);
    int* hb = hslot + m->n_groups + nn + nu;
    for (int gi = 0; gi < m->n_groups; ++gi)
        for (int p = m->grp_ptr[gi]; p < m->grp_ptr[gi + 1]; ++p) hb[m->grp_idx[p]] = hslot[gi];
    cudaError_t e = cudaSuccess;
    int* di = nullptr;
#define GCK(call)                      \
    do {                               \
        e = (call);                    \
        if (e != cudaSuccess) goto err; \
    } while (0)
    GCK(cudaMalloc(&gp->d_arr, sizeof(double) * nd));
    GCK(cudaMemcpy(gp->d_arr, h.data(), sizeof(double) * nd, cudaMemcpyHostToDevice));
    GCK(cudaMalloc(&di, sizeof(int) * hi.size()));
    GCK(cudaMemcpy(di, hi.data(), sizeof(int) * hi.size(), cudaMemcpyHostToDevice));
    GCK(cudaMalloc(&gp->d_scr, sizeof(double) * 10 * nn));
    GCK(cudaMalloc(&gp->col, sizeof(double) * nu));
    GCK(cudaMalloc(&gp->d_flags, sizeof(unsigned)));
    GCK(cudaMemset(gp->d_flags, 0, sizeof(unsigned)));
    GCK(cudaMallocHost(&gp->h_flags, sizeof(unsigned)));
    GCK(cudaMalloc(&gp->d_bits, 2 * sizeof(unsigned long long)));
    GCK(cudaMalloc(&gp->d_nb, sizeof(int)));
#undef GCK
    {
        double* d = gp->d_arr;
        GGeo& g = gp->g;
        g.nel = m->nel;
        g.nq = nq;
        g.NP = NP;
        g.nn = nn;
        g.D = d;
        d += nq * nq;
        g.ar = d;
        g.as = d + 3 * nn;
        g.at = d + 6 * nn;
        g.vert = d + 9 * nn;
        g.Jtv = d + 12 * nn;
        gp->d_w = d + 13 * nn;
        gp->d_wsum = d + 14 * nn;
        g.bproj = gp->d_wsum + m->n_groups;
        d = gp->d_arr + base_bg;
        GRef& r = gp->r;
        r.rho0 = d;
        r.theta0 = d + nn;
        r.P0f = d + 2 * nn;
        r.grho0 = d + 3 * nn;
        r.gth0 = d + 6 * nn;
        r.gvec = d + 9 * nn;
        r.G0 = d + 12 * nn;
        r.H0 = d + 13 * nn;
        r.F0v = d + 14 * nn;
        r.Th0 = d + 17 * nn;
        r.F0c = d + 18 * nn;
        r.Pb = d + 19 * nn;
        r.c0 = d + 20 * nn;
        r.irt0 = d + 21 * nn;
        r.g = rd->g;
        r.R = rd->R;
        r.P0 = rd->P0;
        r.gamma = rd->gamma;
        r.eqset = rd->eqset;
        r.w_zero = wz;
        double cb = 1.0;
        for (int k = 1; k <= 15; ++k) {
            cb = cb * (rd->gamma - (k - 1)) / k;
            r.bc[k - 1] = cb;
        }
        r.bc[15] = 0.0;
        gp->d_gptr = di;
        gp->d_gidx = di + m->n_groups + 1;
        gp->d_gslot = gp->d_gidx + nn;
        gp->d_uid = gp->d_gslot + m->n_groups;
        gp->d_rep = gp->d_uid + nn;
        gp->d_bslot = gp->d_rep + nu;
        g.bslot = gp->d_bslot;
        double* s = gp->d_scr;
        gp->s0 = s;
        gp->s1 = s + nn;
        gp->ua = s + 2 * nn;
        gp->up = s + 5 * nn;
        gp->sP = s + 8 * nn;
        gp->sO = s + 9 * nn;
    }
    *out = gp;
    return HEVI_OK;
err:
    if (di) cudaFree(di);
    hevi_gplan_destroy(gp);
    return fail("general plan allocation", e);
}

int hevi_gplan_destroy(hevi_gplan* gp) {
    if (!gp) return HEVI_OK;
    for (auto& kv : gp->factors) {
        cudaFree(kv.second.A);
        cudaFree(kv.second.band);
        cudaFree(kv.second.LUP);
        cudaFree(kv.second.piv);
    }
    cudaFree(gp->d_arr);
    cudaFree(gp->d_gptr);
    cudaFree(gp->d_scr);
    cudaFree(gp->col);
    cudaFree(gp->d_flags);
    if (gp->h_flags) cudaFreeHost(gp->h_flags);
    cudaFree(gp->d_bits);
    cudaFree(gp->d_nb);
    delete gp;
    return HEVI_OK;
}

int hevi_g_work_fields(const hevi_gplan* gp) { return gp ? 7 : 0; }

int hevi_g_rhs(hevi_gplan* gp, const double* q, double* R, void* stream) {
    if (!gp || !q || !R) return fail("null argument");
    return g_rhs(gp, q, R, 0, (cudaStream_t)stream);
}

int hevi_g_linear_v(hevi_gplan* gp, const double* q, double* L, void* stream) {
    if (!gp || !q || !L) return fail("null argument");
    return g_linear_v(gp, q, L, (cudaStream_t)stream);
}

int hevi_g_factor(hevi_gplan* gp, double lam, int* nb_out, int* pivoted_out, void* stream) {
    if (!gp) return fail("null plan");
    if (!(lam > 0.0)) return fail("implicit solve requires positive lam");
    int rc = g_factor(gp, lam, (cudaStream_t)stream);
    if (rc) return rc;
    const GFactor* f = g_find(gp, lam);
    if (nb_out) *nb_out = f->nb;
    if (pivoted_out) *pivoted_out = f->pivoted;
    return HEVI_OK;
}

int hevi_g_column_matrix(hevi_gplan* gp, double lam, int col, double* A_host, void* stream) {
    const GFactor* f = gp ? g_find(gp, lam) : nullptr;
    if (!f) {
        g_err = "lam not factored";
        return HEVI_ENOFACTOR;
    }
    if (col >= gp->n_col || !A_host) return fail("bad column");
    const size_t MM = (size_t)gp->n_lev * gp->n_lev;
    cudaStream_t st = (cudaStream_t)stream;
    // col < 0: every column (n_col x M x M)
    CK(cudaMemcpyAsync(A_host, f->A + (size_t)(col < 0 ? 0 : col) * MM,
                       sizeof(double) * MM * (col < 0 ? gp->n_col : 1), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return HEVI_OK;
}

int hevi_g_solve(hevi_gplan* gp, double lam, const double* qe, double* q, void* stream) {
    if (!gp || !qe || !q) return fail("null argument");
    if (qe == q) return fail("solve: qe and q must not alias");
    return g_solve(gp, lam, qe, q, (cudaStream_t)stream);
}

int hevi_g_ark2_step(hevi_gplan* gp, double dt, const double* tab, double* Q, double* work, void* stream) {
    if (!gp || !tab || !Q || !work) return fail("null argument");
    cudaStream_t st = (cudaStream_t)stream;
    const double lam = tab[9 + 3 * 1 + 1] * dt;   // problem.lam = tableau.diag * dt
    int rc = g_factor(gp, lam, st);
    if (rc) return rc;
    const long long n5 = 5 * gp->nn;
    double *R0 = work, *L0 = work + n5, *R1 = work + 2 * n5, *L1 = work + 3 * n5, *R2 = work + 4 * n5,
           *P = work + 5 * n5, *Qi = work + 6 * n5;
    const double* a = tab;
    const double* at = tab + 9;
    const double* b = tab + 18;
    // imexcore.py:393-414
    if ((rc = g_rhs(gp, Q, R0, 0, st)) || (rc = g_linear_v(gp, Q, L0, st))) return rc;
    kg_pred<<<blocks_for(n5), 256, 0, st>>>(Q, R0, L0, nullptr, nullptr, 1, dt, a[3], at[3], 0.0, 0.0, P, n5);
    CK(cudaGetLastError());
    if ((rc = g_solve(gp, lam, P, Qi, st))) return rc;
    if ((rc = g_rhs(gp, Qi, R1, 1, st)) || (rc = g_linear_v(gp, Qi, L1, st))) return rc;
    kg_pred<<<blocks_for(n5), 256, 0, st>>>(Q, R0, L0, R1, L1, 2, dt, a[6], at[6], a[7], at[7], P, n5);
    CK(cudaGetLastError());
    if ((rc = g_solve(gp, lam, P, Qi, st))) return rc;
    if ((rc = g_rhs(gp, Qi, R2, 2, st))) return rc;
    kg_final<<<blocks_for(n5), 256, 0, st>>>(Q, R0, R1, R2, dt * b[0], dt * b[1], dt * b[2], Q, n5, gp->d_flags);
    CK(cudaGetLastError());
    return HEVI_OK;
}

int hevi_g_rk35_step(hevi_gplan* gp, double dt, double* Q, double* work, void* stream) {
    if (!gp || !Q || !work) return fail("null argument");
    cudaStream_t st = (cudaStream_t)stream;
    // Shu-Osher SSP RK(5,3) (imexcore.py:81-126), as hevi_rk35_step
    static const double al_a[5] = {0.0, 0.0, 0.355909775063327, 0.367933791638137, 0.237593836598569};
    static const double al_b[5] = {1.0, 1.0, 0.644090224936674, 0.632066208361863, 0.762406163401431};
    static const double be[5] = {0.377268915331368, 0.377268915331368, 0.242995220537396,
                                 0.238458932846290, 0.287632146308408};
    const long long n5 = 5 * gp->nn;
    double* U[4] = {work, work + n5, work + 2 * n5, work + 3 * n5};
    double* R = work + 4 * n5;
    const double* qin[5] = {Q, U[0], U[1], U[2], U[3]};
    const double* xin[5] = {nullptr, nullptr, Q, Q, U[1]};
    double* out[5] = {U[0], U[1], U[2], U[3], Q};
    for (int i = 0; i < 5; ++i) {
        int rc = g_rhs(gp, qin[i], R, i < 2 ? i : 2, st);
        if (rc) return rc;
        GTerms T;
        int k = 0;
        if (xin[i]) {
            T.x[k] = xin[i];
            T.c[k++] = al_a[i];
        }
        T.x[k] = qin[i];
        T.c[k++] = al_b[i];
        T.x[k] = R;
        T.c[k++] = be[i] * dt;
        T.n = k;
        kg_terms<<<blocks_for(n5), 256, 0, st>>>(T, out[i], n5, i == 4, gp->d_flags);
        CK(cudaGetLastError());
    }
    return HEVI_OK;
}

int hevi_g_dss(hevi_gplan* gp, const double* in, double* out, int nf, void* stream) {
    if (!gp || !in || !out || nf < 1) return fail("null argument");
    cudaStream_t st = (cudaStream_t)stream;
    for (int f0 = 0; f0 < nf; f0 += 4) {
        const int k = std::min(4, nf - f0);
        int rc = g_dss(gp, in + f0 * gp->nn, out + f0 * gp->nn, k, 0, st);
        if (rc) return rc;
    }
    return HEVI_OK;
}

int hevi_g_grad(hevi_gplan* gp, int vertical_only, const double* f, double* out, void* stream) {
    if (!gp || !f || !out) return fail("null argument");
    cudaStream_t st = (cudaStream_t)stream;
    if (vertical_only) {
        int rc = g_vgrad(gp, f, st);
        if (rc) return rc;
        kg_times_vert<<<blocks_for(gp->nn), 256, 0, st>>>(gp->g, gp->s0, out);
        CK(cudaGetLastError());
        return HEVI_OK;
    }
    G_DISPATCH(gp->g.nq, { kg_graddiv<NQ><<<gp->g.nel, NQ * NQ * NQ, 0, st>>>(gp->g, f, 0, out); });
    CK(cudaGetLastError());
    return g_dss(gp, out, out, 3, 0, st);
}

int hevi_g_div(hevi_gplan* gp, int vertical_only, const double* vec, double* out, void* stream) {
    if (!gp || !vec || !out) return fail("null argument");
    cudaStream_t st = (cudaStream_t)stream;
    if (vertical_only) {
        GVArgs a = {};
        a.vec = const_cast<double*>(vec);
        a.d0 = out;
        int rc = g_vderiv(gp, a, 3, st);
        return rc ? rc : g_dss(gp, out, out, 1, 0, st);
    }
    G_DISPATCH(gp->g.nq, { kg_graddiv<NQ><<<gp->g.nel, NQ * NQ * NQ, 0, st>>>(gp->g, vec, 1, out); });
    CK(cudaGetLastError());
    return g_dss(gp, out, out, 1, 0, st);
}

int hevi_g_flags(hevi_gplan* gp, unsigned* flags, int reset, void* stream) {
    if (!gp || !flags) return fail("null argument");
    return g_flags_now(gp, flags, reset, (cudaStream_t)stream);
}

// ---- 3D-IMEX pieces (ImplicitProblem dim = "3d" / "1d" Krylov path) --------
int hevi_g_schur3_ua(hevi_gplan* gp, double lam, const double* qe, double* ua, double* Pe, void* stream) {
    if (!gp || !qe || !ua || !Pe) return fail("null argument");
    kg_schur_ua<<<blocks_for(gp->nn), 256, 0, (cudaStream_t)stream>>>(gp->g, gp->r, qe, lam, ua, Pe, gp->d_flags);
    CK(cudaGetLastError());
    return HEVI_OK;
}

int hevi_g_schur3_up(hevi_gplan* gp, double lam, int vertical_only, const double* P, double* up, void* stream) {
    if (!gp || !P || !up) return fail("null argument");
    cudaStream_t st = (cudaStream_t)stream;
    int rc;
    if (vertical_only) {
        if ((rc = g_vgrad(gp, P, st))) return rc;
        kg_up<<<blocks_for(gp->nn), 256, 0, st>>>(gp->g, gp->r, P, gp->s0, lam, up, gp->d_flags);
    } else {
        G_DISPATCH(gp->g.nq, { kg_graddiv<NQ><<<gp->g.nel, NQ * NQ * NQ, 0, st>>>(gp->g, P, 0, gp->up); });
        CK(cudaGetLastError());
        if ((rc = g_dss(gp, gp->up, gp->up, 3, 0, st))) return rc;
        kg_up3<<<blocks_for(gp->nn), 256, 0, st>>>(gp->g, gp->r, P, gp->up, lam, up, gp->d_flags);
    }
    CK(cudaGetLastError());
    return HEVI_OK;
}

int hevi_g_schur3_flux(hevi_gplan* gp, double lam, int vertical_only, const double* P, const double* vel,
                       double* out, void* stream) {
    if (!gp || !P || !vel || !out) return fail("null argument");
    cudaStream_t st = (cudaStream_t)stream;
    int rc;
    if (vertical_only) {
        GVArgs a = {};
        a.vec = const_cast<double*>(vel);
        a.d0 = gp->s1;
        if ((rc = g_vderiv(gp, a, 3, st))) return rc;
    } else {
        G_DISPATCH(gp->g.nq, { kg_graddiv<NQ><<<gp->g.nel, NQ * NQ * NQ, 0, st>>>(gp->g, vel, 1, gp->s1); });
        CK(cudaGetLastError());
    }
    if ((rc = g_dss(gp, gp->s1, gp->s1, 1, 0, st))) return rc;
    kg_lhs<<<blocks_for(gp->nn), 256, 0, st>>>(gp->g, gp->r, P, vel, gp->s1, lam, out);
    CK(cudaGetLastError());
    return HEVI_OK;
}

int hevi_g_schur3_extract(hevi_gplan* gp, double lam, int vertical_only, const double* P, const double* ua,
                          const double* up, const double* qe, double* q, void* stream) {
    if (!gp || !P || !ua || !up || !qe || !q) return fail("null argument");
    kg_extract3<<<blocks_for(gp->nn), 256, 0, (cudaStream_t)stream>>>(gp->g, gp->r, P, ua, up, qe, lam,
                                                                      vertical_only, q);
    CK(cudaGetLastError());
    return HEVI_OK;
}

int hevi_g_linear3(hevi_gplan* gp, const double* q, double* out, void* stream) {
    if (!gp || !q || !out) return fail("null argument");
    cudaStream_t st = (cudaStream_t)stream;
    kg_plin<<<blocks_for(gp->nn), 256, 0, st>>>(gp->g, gp->r, q, gp->sP);
    CK(cudaGetLastError());
    G_DISPATCH(gp->g.nq, {
        kg_graddiv<NQ><<<gp->g.nel, NQ * NQ * NQ, 0, st>>>(gp->g, gp->sP, 0, gp->up);
        kg_graddiv<NQ><<<gp->g.nel, NQ * NQ * NQ, 0, st>>>(gp->g, q + gp->nn, 1, gp->s1);
    });
    CK(cudaGetLastError());
    int rc;
    if ((rc = g_dss(gp, gp->up, gp->up, 3, 0, st)) || (rc = g_dss(gp, gp->s1, gp->s1, 1, 0, st))) return rc;
    kg_lin3<<<blocks_for(gp->nn), 256, 0, st>>>(gp->g, gp->r, q, gp->up, gp->s1, out);
    CK(cudaGetLastError());
    return HEVI_OK;
}

int hevi_g_dot(hevi_gplan* gp, const double* x, const double* y, long long n, double* out_host, void* stream) {
    if (!gp || !x || !y || !out_host) return fail("null argument");
    cudaStream_t st = (cudaStream_t)stream;
    double* part = gp->sO;   // KV_BLOCKS partials (scratch) and the sum after them
    if (gp->nn < KV_BLOCKS + 1) return fail("general plan too small for the dot scratch");
    kg_dot<<<KV_BLOCKS, KV_T, 0, st>>>(x, y, n, part);
    k3_sum<<<1, 32, 0, st>>>(part, KV_BLOCKS, part + KV_BLOCKS);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out_host, part + KV_BLOCKS, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return HEVI_OK;
}
