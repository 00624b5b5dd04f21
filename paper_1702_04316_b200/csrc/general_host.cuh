// general_host.cuh -- launch sequences of the general-mesh path (included by
// hevi.cu inside its second anonymous namespace, after blocks_for).
#pragma once

// element kernels are templated on nq = N + 1 (one CTA per element)
#define G_DISPATCH(NQV, ...)                                          \
    switch (NQV) {                                                    \
        case 2: { constexpr int NQ = 2; __VA_ARGS__; } break;         \
        case 3: { constexpr int NQ = 3; __VA_ARGS__; } break;         \
        case 4: { constexpr int NQ = 4; __VA_ARGS__; } break;         \
        case 5: { constexpr int NQ = 5; __VA_ARGS__; } break;         \
        case 6: { constexpr int NQ = 6; __VA_ARGS__; } break;         \
        case 7: { constexpr int NQ = 7; __VA_ARGS__; } break;         \
        case 8: { constexpr int NQ = 8; __VA_ARGS__; } break;         \
        case 9: { constexpr int NQ = 9; __VA_ARGS__; } break;         \
        default: return fail("general mesh: order outside 1..8");     \
    }

int g_dss(const hevi_gplan* gp, const double* in, double* out, int nf, int proj, cudaStream_t st) {
    kg_dss<<<blocks_for(gp->n_groups), 256, 0, st>>>(gp->d_gptr, gp->d_gidx, gp->d_w, gp->d_wsum, gp->d_gslot,
                                                     gp->g.bproj, in, out, nf, gp->nn, gp->n_groups, proj);
    CK(cudaGetLastError());
    return HEVI_OK;
}

int g_rhs(const hevi_gplan* gp, const double* q, double* R, int stage, cudaStream_t st) {
    const size_t smem = sizeof(double) * (gp->r.eqset ? 15 : 6) * gp->g.NP;
    G_DISPATCH(gp->g.nq, {
        auto k = kg_rhs<NQ>;
        if (smem > 48 * 1024) CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k<<<gp->g.nel, NQ * NQ * NQ, smem, st>>>(gp->g, gp->r, q, R, gp->d_flags, stage);
    });
    CK(cudaGetLastError());
    return g_dss(gp, R, R, 5, 1, st);
}

int g_vderiv(const hevi_gplan* gp, const GVArgs& a, int kind, cudaStream_t st) {
    G_DISPATCH(gp->g.nq, { kg_vderiv<NQ><<<gp->g.nel, NQ * NQ * NQ, 0, st>>>(gp->g, gp->r, a, kind); });
    CK(cudaGetLastError());
    return HEVI_OK;
}

int g_linear_v(const hevi_gplan* gp, const double* q, double* L, cudaStream_t st) {
    GVArgs a = {};
    a.q = q;
    a.d0 = gp->s0;
    a.d1 = gp->s1;
    int rc = g_vderiv(gp, a, 0, st);
    if (!rc) rc = g_dss(gp, gp->s0, gp->s0, 2, 0, st);
    if (rc) return rc;
    kg_lv<<<blocks_for(gp->nn), 256, 0, st>>>(gp->g, gp->r, q, gp->s0, gp->s1, L);
    CK(cudaGetLastError());
    return HEVI_OK;
}

// rhs_schur_build: ua -> gp->ua, Schur RHS -> rhs
int g_schur_rhs(const hevi_gplan* gp, double lam, const double* qe, double* rhs, cudaStream_t st) {
    GVArgs a = {};
    a.q = qe;
    a.vec = gp->ua;
    a.d0 = gp->s0;
    a.lam = lam;
    a.flags = gp->d_flags;
    int rc = g_vderiv(gp, a, 1, st);
    if (!rc) rc = g_dss(gp, gp->s0, gp->s0, 1, 0, st);
    if (rc) return rc;
    kg_schur_rhs<<<blocks_for(gp->nn), 256, 0, st>>>(gp->g, gp->r, qe, gp->ua, gp->s0, lam, rhs);
    CK(cudaGetLastError());
    return HEVI_OK;
}

// DSS(Jtv dt x) -> gp->s0
int g_vgrad(const hevi_gplan* gp, const double* x, cudaStream_t st) {
    GVArgs a = {};
    a.x = x;
    a.d0 = gp->s0;
    int rc = g_vderiv(gp, a, 2, st);
    return rc ? rc : g_dss(gp, gp->s0, gp->s0, 1, 0, st);
}

// lhs_schur(P) (imexcore.py:270-271) -> out
int g_lhs(const hevi_gplan* gp, double lam, const double* P, double* out, cudaStream_t st) {
    int rc = g_vgrad(gp, P, st);
    if (rc) return rc;
    kg_up<<<blocks_for(gp->nn), 256, 0, st>>>(gp->g, gp->r, P, gp->s0, lam, gp->up, gp->d_flags);
    CK(cudaGetLastError());
    GVArgs a = {};
    a.vec = gp->up;
    a.d0 = gp->s1;
    if ((rc = g_vderiv(gp, a, 3, st))) return rc;
    if ((rc = g_dss(gp, gp->s1, gp->s1, 1, 0, st))) return rc;
    kg_lhs<<<blocks_for(gp->nn), 256, 0, st>>>(gp->g, gp->r, P, gp->up, gp->s1, lam, out);
    CK(cudaGetLastError());
    return HEVI_OK;
}

const GFactor* g_find(const hevi_gplan* gp, double lam) {
    auto it = gp->factors.find(lam_key(lam));
    return it == gp->factors.end() ? nullptr : &it->second;
}

int g_factor(hevi_gplan* gp, double lam, cudaStream_t st) {
    if (g_find(gp, lam)) return HEVI_OK;
    const int nc = gp->n_col, M = gp->n_lev;
    const long long nn = gp->nn;
    GFactor f;
    f.lam = lam;
    CK(cudaMalloc(&f.A, sizeof(double) * (size_t)nc * M * M));
    double* P = gp->sP;
    double* out = gp->sO;
    for (int lev = 0; lev < M; ++lev) {
        kg_probe_vec<<<blocks_for(nn), 256, 0, st>>>(gp->d_uid, M, lev, -1, P, nn);
        CK(cudaGetLastError());
        int rc = g_lhs(gp, lam, P, out, st);
        if (rc) return rc;
        kg_probe_store<<<blocks_for((long long)nc * M), 256, 0, st>>>(out, gp->d_rep, nc, M, lev, f.A);
        CK(cudaGetLastError());
    }
    // sampled cross-column leakage check (columnsolve.py:94-101): probe one
    // column alone, nothing may reach another column
    {
        kg_probe_vec<<<blocks_for(nn), 256, 0, st>>>(gp->d_uid, M, M / 2, 0, P, nn);
        CK(cudaGetLastError());
        int rc = g_lhs(gp, lam, P, out, st);
        if (rc) return rc;
        kg_gather<<<blocks_for((long long)nc * M), 256, 0, st>>>(out, gp->d_rep, gp->col, (long long)nc * M);
        CK(cudaMemsetAsync(gp->d_bits, 0, 2 * sizeof(unsigned long long), st));
        kg_absmax_bits<<<1, 256, 0, st>>>(gp->col, M, M, M, gp->d_bits);
        kg_absmax_bits<<<blocks_for((long long)nc * M), 256, 0, st>>>(gp->col, (long long)nc * M, 0, M,
                                                                       gp->d_bits + 1);
        CK(cudaGetLastError());
        unsigned long long h[2];
        CK(cudaMemcpyAsync(h, gp->d_bits, sizeof(h), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        double own, other;
        memcpy(&own, &h[0], 8);
        memcpy(&other, &h[1], 8);
        if (other > 1e-13 * std::max(1.0, own)) {
            cudaFree(f.A);
            return fail("cross-column leakage detected in the vertical operator; columns are not independent");
        }
    }
    // bandwidth of the probed pattern and the no-pivot banded LU
    CK(cudaMemsetAsync(gp->d_bits, 0, sizeof(unsigned long long), st));
    kg_absmax_bits<<<blocks_for((long long)nc * M * M), 256, 0, st>>>(f.A, (long long)nc * M * M, 0, 0, gp->d_bits);
    CK(cudaMemsetAsync(gp->d_nb, 0, sizeof(int), st));
    kg_bandwidth<<<blocks_for((long long)nc * M * M), 256, 0, st>>>(f.A, nc, M, gp->d_bits, gp->d_nb);
    CK(cudaGetLastError());
    unsigned long long sb = 0;
    CK(cudaMemcpyAsync(&sb, gp->d_bits, sizeof(sb), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&f.nb, gp->d_nb, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    double norm;
    memcpy(&norm, &sb, 8);
    const int W = 2 * f.nb - 1;
    CK(cudaMalloc(&f.band, sizeof(double) * (size_t)nc * M * W));
    k_band_pack<<<blocks_for((long long)nc * M * W), 256, 0, st>>>(f.A, f.band, nc, M, f.nb);
    int* d_bad;
    CK(cudaMallocAsync(&d_bad, sizeof(int), st));
    const int big = 0x7fffffff;
    CK(cudaMemcpyAsync(d_bad, &big, sizeof(int), cudaMemcpyHostToDevice, st));
    k_band_lu<<<(nc + 127) / 128, 128, 0, st>>>(f.band, nc, M, f.nb, norm, d_bad);
    CK(cudaGetLastError());
    int bad = big;
    CK(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(d_bad, st));
    CK(cudaStreamSynchronize(st));
    if (bad != big) {
        // factor_with_fallback (columnsolve.py:141-153): pivoted dense LU of every column
        CK(cudaMalloc(&f.LUP, sizeof(double) * (size_t)nc * M * M));
        CK(cudaMalloc(&f.piv, sizeof(int) * (size_t)nc * M));
        CK(cudaMemcpyAsync(f.LUP, f.A, sizeof(double) * (size_t)nc * M * M, cudaMemcpyDeviceToDevice, st));
        int* d_info;
        CK(cudaMallocAsync(&d_info, sizeof(int) * nc, st));
        k_lu_pivot_batched<<<nc, 256, 0, st>>>(f.LUP, f.piv, M, d_info);
        CK(cudaGetLastError());
        CK(cudaFreeAsync(d_info, st));
        f.pivoted = 1;
    }
    gp->factors.emplace(lam_key(lam), f);
    return HEVI_OK;
}

// columnsolve.solve_direct (:191-210): Schur RHS, gather, per-column
// substitution, scatter, extraction
int g_solve(hevi_gplan* gp, double lam, const double* qe, double* q, cudaStream_t st) {
    const GFactor* f = g_find(gp, lam);
    if (!f) {
        g_err = "lam not factored";
        return HEVI_ENOFACTOR;
    }
    const int nc = gp->n_col, M = gp->n_lev;
    int rc = g_schur_rhs(gp, lam, qe, gp->sP, st);
    if (rc) return rc;
    kg_gather<<<blocks_for((long long)nc * M), 256, 0, st>>>(gp->sP, gp->d_rep, gp->col, (long long)nc * M);
    if (f->pivoted)
        k_lu_pivot_solve<<<(nc + 127) / 128, 128, 0, st>>>(f->LUP, f->piv, gp->col, nc, M);
    else
        k_band_solve<<<(nc + 127) / 128, 128, 0, st>>>(f->band, gp->col, nc, M, f->nb);
    kg_scatter<<<blocks_for(gp->nn), 256, 0, st>>>(gp->col, gp->d_uid, gp->sP, gp->nn);
    CK(cudaGetLastError());
    if ((rc = g_vgrad(gp, gp->sP, st))) return rc;
    kg_extract<<<blocks_for(gp->nn), 256, 0, st>>>(gp->g, gp->r, gp->sP, gp->s0, gp->ua, qe, lam, q, gp->d_flags);
    CK(cudaGetLastError());
    return HEVI_OK;
}

int g_flags_now(hevi_gplan* gp, unsigned* out, int reset, cudaStream_t st) {
    CK(cudaMemcpyAsync(gp->h_flags, gp->d_flags, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    if (reset) CK(cudaMemsetAsync(gp->d_flags, 0, sizeof(unsigned), st));
    CK(cudaStreamSynchronize(st));
    *out = gp->h_flags[0];
    return HEVI_OK;
}
