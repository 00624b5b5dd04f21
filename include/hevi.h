/*
 * hevi.h -- C ABI of the B200-native HEVI 1D-IMEX ARK2 step (libhevi.so).
 *
 * The reference (dycore, pure Python/NumPy) has no FFI for this path; its
 * drop-in boundary is the Python call protocol listed in SURVEY.md 8(b).
 * Each entry point below replaces one reference function; the Python layer
 * paper_1702_04316_b200 rebinds the reference protocol on top of it.
 *
 * Conventions
 *   - all pointers to state/work arrays are DEVICE pointers to fp64
 *     "lattice" arrays: field-major, field f at  f*fs + (gz*lY + iy)*px + ix
 *     (ix, iy local to the rank window; gz = level); fs = Z*lY*px.
 *     Fields: 0 rho', 1 u, 2 v, 3 w, 4 theta' (euler.py:39-58, set2nc).
 *   - E-vector arrays use the reference layout (5, nel, nqt, nqs, nqr)
 *     with element e = (kz*ney + ky)*nex + kx (specgrid.py:185-201).
 *   - `stream` is a cudaStream_t passed as void*.
 *   - return value: HEVI_OK (0) or a negative HEVI_E* code; no C++
 *     exception crosses the ABI.  Numerical failures detected on the
 *     device are sticky flags read back with hevi_flags().
 */
#ifndef HEVI_H
#define HEVI_H

#ifdef __cplusplus
extern "C" {
#endif

#define HEVI_OK 0
#define HEVI_EARG (-1)        /* bad argument / unsupported configuration */
#define HEVI_ECUDA (-2)       /* CUDA runtime error (see hevi_last_error) */
#define HEVI_ENOFACTOR (-3)   /* solve requested for an unfactored lam */

/* device flag bits (hevi_flags); stage s = 0,1,2 are the three explicit
 * evaluations of an ARK2 step (a single rhs() call reports as stage 0) */
#define HEVI_F_NONFINITE_IN(s) (1u << ((s) * 4 + 0)) /* euler.py:445-446 FloatingPointError */
#define HEVI_F_EOS(s) (1u << ((s) * 4 + 1))          /* euler.py:183-184 ValueError */
#define HEVI_F_NONFINITE_OUT (1u << 12)              /* imexcore.py:412-413 FloatingPointError */
#define HEVI_F_PIVOT (1u << 13)                      /* columnsolve.py:135-137 RuntimeError */
#define HEVI_F_AINV (1u << 14)                       /* imexcore.py:214-215 FloatingPointError */

typedef struct hevi_plan hevi_plan;

/* Structured box (specgrid.build_box_mesh slab, or the SURVEY 8(c) 3D box).
 * Global lattice X = nex*N+1, Y = ney*Ny+1, Z = nez*N+1. */
typedef struct {
    int nex, ney, nez;      /* global element counts                        */
    int N, Ny;              /* polynomial order (Ny = N in 3D, 1 for slab)  */
    int slab;               /* 1: columns keyed by x only (specgrid.py:203) */
    int x0, y0, lX, lY;     /* this rank's lattice window (global origin)   */
    int px;                 /* x pitch of lattice arrays, >= lX             */
    int ex_b, ex_e;         /* owned element range in x  [ex_b, ex_e)       */
    int ey_b, ey_e;         /* owned element range in y                     */
} hevi_grid_desc;

/* Host arrays copied into the plan at creation.  Level tables have length
 * Z and carry the reference-state coefficients of euler.py:70-150 sampled
 * per level; cx/cy/cz are the DSS-averaged metric factors per lattice index
 * (1/dxdr for element-interior points, 1/(dxdr_left + dxdr_right) on
 * element faces); Dx/Dy/Dz are (N+1)^2 / (Ny+1)^2 LGL derivative matrices. */
typedef struct {
    const double *rho0, *theta0, *P0f, *drho0, *dtheta0;
    const double *G0, *H0, *F0z, *rho0G0;
    const double *Pb;       /* EOS(rho0, theta0) per level: euler.equation_of_state
                               of the background, the reference point of the
                               P' = P - P0f evaluation (euler.py:454-457)      */
    const double *cx, *cy, *cz;
    const double *Dx, *Dy, *Dz;
    const double *Theta0, *F0c; /* set2c: rho0 theta0 and gamma P0f / Theta0 (euler.py:103-113) */
    double g, R, P0, gamma;
    int eqset;              /* 0: set2nc (rho', u, v, w, theta'); 1: set2c (rho', U, V, W, Theta') */
} hevi_ref_desc;

int hevi_plan_create(hevi_plan **plan, const hevi_grid_desc *grid, const hevi_ref_desc *ref);
int hevi_plan_destroy(hevi_plan *plan);
const char *hevi_last_error(void);
/* number of doubles in one 5-field lattice array of this plan */
long long hevi_state_size(const hevi_plan *plan);

/* columnsolve.get_factors + factor_with_fallback (columnsolve.py:141-153,
 * 184-188): probe the Schur column operator lhs_schur (imexcore.py:270-271)
 * on the device, no-pivot banded LU (columnsolve.py:111-138), cached per
 * round(lam, 12).  nb_out (may be NULL) receives the detected bandwidth. */
int hevi_factor(hevi_plan *plan, double lam, int *nb_out, void *stream);
/* copy the dense probed column matrix / its LU (M*M, row-major) to host */
int hevi_column_matrix(hevi_plan *plan, double lam, double *A_host, double *LU_host, void *stream);

/* euler.nonlinear_rhs, cG set2nc (euler.py:438-497): R = R(q) */
int hevi_rhs(hevi_plan *plan, const double *q, double *R, void *stream);
/* euler.vertical_restriction (euler.py:368-371): L = L_V(q) */
int hevi_linear_v(hevi_plan *plan, const double *q, double *L, void *stream);
/* ImplicitProblem.solve, direct branch (imexcore.py:312-322 ->
 * columnsolve.solve_direct :191-210): q = (I - lam L_V)^{-1} q_e */
int hevi_solve(hevi_plan *plan, double lam, const double *qe, double *q, void *stream);

/* One explicit stage of the fused ARK2 schedule:
 *   stage 0: reads Q;          writes P(0,3,4), Q1(1,2), A, F
 *   stage 1: reads Q1, A, F;   writes P(0,3,4), A(1,2), F
 *   stage 2: reads A, F;       writes Q
 * work = 4 consecutive lattice arrays [Q1 | A | F | P].
 * tab = {a[3][3], at[3][3], b[3]} row-major (imexcore.py:44-63). */
int hevi_stage(hevi_plan *plan, int stage, double dt, const double *tab,
               double *Q, double *work, void *stream);
/* column solve of a stage: P(0,3,4) -> dst(0,3,4); stage 0 -> Q1, stage 1 -> A */
int hevi_stage_solve(hevi_plan *plan, int stage, double lam, double *work, void *stream);
/* imexcore.ark_imex_step (imexcore.py:385-414), single rank: Q <- step(Q) */
int hevi_ark2_step(hevi_plan *plan, double dt, const double *tab, double *Q, double *work,
                   void *stream);
/* As hevi_ark2_step; with flags & HEVI_STEP_PP_VALID the caller asserts that
 * work's Q1 field 0 holds P'(Q) (euler.py:454-457), as the previous step's
 * stage 2 writes it when hevi_step_chains_pp(plan) is 1, so stage 0 does not
 * form it again.  Steady stepping (cli.py:224-241 hot loop) sets the flag
 * after hevi_pp_refresh once per externally supplied state. */
#define HEVI_STEP_PP_VALID 1u
int hevi_ark2_step_ex(hevi_plan *plan, double dt, const double *tab, double *Q, double *work,
                      unsigned flags, void *stream);
/* hevi_stage with the HEVI_STEP_PP_VALID contract of hevi_ark2_step_ex (stage 0)
 * and, for partitioned runs, the tile subset: HEVI_STAGE_INTERIOR evaluates
 * only the tiles that read no halo point a neighbour rank provides (it may
 * run while the halo exchange is in flight), HEVI_STAGE_BOUNDARY the rest
 * and the domain-end planes (after the exchange); the two calls together
 * are the stage, bitwise.  Paths without the tile split do the whole stage
 * in the boundary call. */
#define HEVI_STAGE_INTERIOR 2u
#define HEVI_STAGE_BOUNDARY 4u
int hevi_stage_ex(hevi_plan *plan, int stage, double dt, const double *tab,
                  double *Q, double *work, unsigned flags, void *stream);
/* tiles of the column-sweep stage kernels in the interior / boundary subsets */
int hevi_stage_tiles(const hevi_plan *plan, int *n_interior, int *n_boundary);
/* P'(Q) into work's Q1 field 0 (the plane the chained step reads) */
int hevi_pp_refresh(hevi_plan *plan, const double *Q, double *work, void *stream);
/* 1 if hevi_ark2_step_ex writes P'(Q^{n+1}) for the next step on this plan */
int hevi_step_chains_pp(const hevi_plan *plan);

/* imexcore.rk35_step (imexcore.py:111-126): SSP RK(5,3) explicit step,
 * Q <- step(Q); work = 4 lattice arrays.  The explicit reference the HEVI
 * step is compared with (BASELINE config 2). */
int hevi_rk35_step(hevi_plan *plan, double dt, double *Q, double *work, void *stream);

/* E-vector <-> lattice (exact for DSS-continuous fields; the lattice takes
 * the first-occurrence copy, columnsolve.unique_space rep :28-34) */
int hevi_evec_to_lattice(hevi_plan *plan, const double *E, double *Lat, int nfields, void *stream);
int hevi_lattice_to_evec(hevi_plan *plan, const double *Lat, double *E, int nfields, void *stream);
/* specgrid.apply_dss / apply_dss_many (specgrid.py:535-548) on E-vectors
 * (nfields stacked): every coincident node copy <- sum_c w_c f_c / sum_c w_c,
 * w = wJ per node as the product of per-axis tables wx[kx*(N+1)+i] (GLL
 * weight x half element width), wy, wz (device arrays).  Whole-domain
 * plans only; Ein and Eout must not alias. */
int hevi_dss(hevi_plan *plan, const double *Ein, double *Eout, int nfields, const double *wx,
             const double *wy, const double *wz, void *stream);

/* sticky device flags: OR of HEVI_F_* since the last reset (synchronises stream) */
int hevi_flags(hevi_plan *plan, unsigned *flags, int reset, void *stream);

/* Generic batched column API on per-column banded storage, the reference's
 * ColumnJacobian path for arbitrary (n_col, M, M) matrices:
 *   band layout: band[(d*M + k)*n_col + c], d = j - k + nb - 1 in [0, 2nb-2]
 * hevi_band_pack:  dense (n_col, M, M) row-major -> band
 * hevi_band_lu:    columnsolve.lu_factor_banded (:111-138), in place;
 *                  *bad_col receives the first degenerate column or -1
 * hevi_band_solve: columnsolve.solve_columns_direct (:156-181), rhs (n_col, M)
 *                  row-major, solved in place                                  */
/* 3D-IMEX pressure (Schur) form, dim = "3d" (imexcore.py:200-298), and the
 * full linear operator (euler.linear_operator, vertical_only=False,
 * euler.py:313-365), on lattice arrays of this plan (vectors of 3 fields:
 * ua, up, vel; field stride = the plan's):
 *   hevi_linear3         out = L(q), 5 fields
 *   hevi_schur3_up       up = ImplicitProblem._up(P)                (:245-257)
 *   hevi_schur3_flux     out = P - _helmholtz_flux(vel)             (:259-268)
 *                        (lhs_schur with vel = up; the Schur rhs with P = Pe, vel = ua)
 *   hevi_schur3_ua       ua, Pe of rhs_schur_build                  (:229-243)
 * vertical_only != 0 gives the dim = "1d" operators (grad_vc / div_vc,
 * euler.py:292-300) for Krylov solves of the 1D form.
 *   hevi_schur3_extract  q = extract_from_pressure(P, ua, q_e), up = _up(P)  (:273-298)
 * Krylov vector kernels (krylov.py): hevi_wdot = the E-vector dot product of
 * two continuous lattice states of nf fields (multiplicity-weighted,
 * deterministic order);
 * hevi_axpby: y = alpha x + beta y over n doubles. */
int hevi_linear3(hevi_plan *plan, const double *q, double *out, void *stream);
/* Discretization.gradc / grad_vc (euler.py:281-295): out (3 lattice fields)
 * = DSS-projected gradient of the scalar lattice field f; vertical_only = 1
 * gives grad_vc (x, y components zero on a box, vert = z) */
int hevi_grad(hevi_plan *plan, int vertical_only, const double *f, double *out, void *stream);
/* Discretization.divc / div_vc (euler.py:287-300): out = DSS-projected
 * divergence of the 3-field lattice vector vec (vertical_only: d/dz of vec_z) */
int hevi_div(hevi_plan *plan, int vertical_only, const double *vec, double *out, void *stream);
int hevi_schur3_up(hevi_plan *plan, double lam, int vertical_only, const double *P, double *up,
                   void *stream);
int hevi_schur3_flux(hevi_plan *plan, double lam, int vertical_only, const double *P,
                     const double *vel, double *out, void *stream);
int hevi_schur3_ua(hevi_plan *plan, double lam, const double *qe, double *ua, double *Pe, void *stream);
int hevi_schur3_extract(hevi_plan *plan, double lam, const double *P, const double *ua,
                        const double *up, const double *qe, double *q, void *stream);
int hevi_wdot(const hevi_plan *plan, const double *x, const double *y, int nf, double *out_host,
              void *stream);
int hevi_axpby(long long n, double alpha, const double *x, double beta, double *y, void *stream);

/* Direct solve of the standard 5-variable form (columnsolve.solve_direct with
 * form = "standard", columnsolve.py:196-204) on lattice arrays of this plan:
 * q = (I - lam L_V)^-1 q_e column by column with one shared band LU factor
 * (band storage of hevi_band_pack with n_col = 1, M = 5 Z, unknown lev*5 + field). */
int hevi_std_solve(const hevi_plan *plan, const double *band, int M, int nb, const double *qe,
                   double *q, void *stream);

/* Halo exchange of the column-partitioned step (SURVEY 8(b) "halo_pack"): copy
 * the region [xlo, xhi) x [ylo, yhi) (global lattice indices, all levels, nf
 * fields) of a lattice array of this plan into / out of a contiguous
 * (nf, Z, yhi-ylo, xhi-xlo) buffer for one NCCL send / recv per neighbour. */
int hevi_halo_pack(const hevi_plan *plan, const double *q, int nf, int xlo, int xhi, int ylo,
                   int yhi, double *buf, void *stream);
int hevi_halo_unpack(const hevi_plan *plan, double *q, int nf, int xlo, int xhi, int ylo, int yhi,
                     const double *buf, void *stream);

/* Run diagnostics (bench.total_mass / max_perturbations, bench.py:131-137) of a
 * lattice state of this plan: out_host[0] = sum_g Wx[gx] Wy[gy] Wz[gz] (rho0 +
 * rho'), out_host[1] = max |rho'|, out_host[2] = max |q4|; Wx/Wy/Wz are the
 * per-axis unique-point quadrature weights (device arrays of X, Y, Z). */
int hevi_diagnostics(const hevi_plan *plan, const double *q, const double *wx, const double *wy,
                     const double *wz, double *out_host, void *stream);

/* columnsolve.factor_with_fallback (columnsolve.py:141-153) pivoted path:
 * hevi_lu_pivot:       batched in-place partial-pivoting LU of (n_col, M, M)
 *                      row-major matrices (scipy.linalg.lu_factor / getrf:
 *                      piv[c*M+k] = row interchanged with k, 0-based;
 *                      info_host[c] = k+1 for the first exactly-zero pivot)
 * hevi_lu_pivot_solve: scipy.linalg.lu_solve per column, rhs (n_col, M) in place */
int hevi_lu_pivot(double *A, int *piv, int n_col, int M, int *info_host, void *stream);
int hevi_lu_pivot_solve(const double *LU, const int *piv, double *rhs, int n_col, int M, void *stream);

/* plan options; HEVI_OPT_FORCE_PIVOTED makes hevi_factor keep the pivoted
 * dense factor even when the no-pivot LU succeeds (exercises the fallback) */
#define HEVI_OPT_FORCE_PIVOTED 1
int hevi_plan_set_option(hevi_plan *plan, int option, int value);
/* whether the factor of lam took the pivoted fallback (columnsolve.py:150-152) */
int hevi_factor_pivoted(const hevi_plan *plan, double lam, int *pivoted);

int hevi_band_pack(const double *dense, double *band, int n_col, int M, int nb, void *stream);
int hevi_band_unpack(const double *band, double *dense, int n_col, int M, int nb, void *stream);
int hevi_band_lu(double *band, int n_col, int M, int nb, double norm, int *bad_col, void *stream);
int hevi_band_solve(const double *band, double *rhs, int n_col, int M, int nb, void *stream);
/* max |a_i| over n doubles (device), deterministic */
int hevi_absmax(const double *a, long long n, double *out_host, void *stream);

/* ---------------------------------------------------------------------------
 * General curvilinear element meshes (the cubed-sphere shell,
 * specgrid.build_cubed_sphere_mesh, specgrid.py:257-306): the same path on
 * the reference's own E-vector layout (nf, nel, nq, nq, nq), nn = nel*nq^3
 * nodes, node n = ((e*nq + k)*nq + j)*nq + i.  Vector fields are
 * component-major [3][nn].  Columns have their own Schur factors
 * (columnsolve.build_column_jacobian per column, :75-108).
 * ------------------------------------------------------------------------- */
typedef struct hevi_gplan hevi_gplan;

/* host arrays, copied at creation (metric terms of specgrid.compute_metrics,
 * :404-455; DSS groups of build_dss_map, :523-532; projectors of
 * euler.boundary_projectors, :218-258; unique space of columnsolve.unique_space) */
typedef struct {
    int nel, N;
    const double *D;                 /* (N+1)^2 LGL derivative, row-major      */
    const double *ar, *as, *at;      /* contravariant a^r, a^s, a^t [3][nn]     */
    const double *vert;              /* radial unit vector [3][nn]              */
    const double *Jtv;               /* a^t . vert [nn]                         */
    const double *w;                 /* wJ per node [nn]                        */
    int n_groups;
    const int *grp_ptr, *grp_idx;    /* CSR: members of each group, flat-node order */
    const double *grp_wsum;          /* sum of wJ per group                     */
    int n_proj;
    const int *grp_slot;             /* per group: projector index or -1        */
    const double *proj;              /* [n_proj][3][3] tangential projectors    */
    int n_col, n_lev;
    const int *uid;                  /* node -> col*n_lev + lev                 */
    const int *rep;                  /* unique point -> first node              */
} hevi_gmesh_desc;

/* per-node background (euler.ReferenceState, euler.py:70-177) */
typedef struct {
    const double *rho0, *theta0, *P0f;       /* [nn]                  */
    const double *grad_rho0, *grad_theta0;   /* [3][nn]               */
    const double *gvec;                      /* g * vert [3][nn]      */
    const double *G0, *H0;                   /* set2nc gamma P0f/rho0, gamma P0f/theta0 */
    const double *F0vec;                     /* [3][nn] G0 grad rho0 + H0 grad theta0  */
    const double *Theta0, *F0c;              /* set2c rho0 theta0, gamma P0f/Theta0     */
    const double *Pb;                        /* EOS(rho0, theta0) [nn]                  */
    double g, R, P0, gamma;
    int eqset;                               /* 0 set2nc, 1 set2c */
} hevi_gref_desc;

int hevi_gplan_create(hevi_gplan **plan, const hevi_gmesh_desc *mesh, const hevi_gref_desc *ref);
int hevi_gplan_destroy(hevi_gplan *plan);
/* E-vectors of the plan's work area used by hevi_g_ark2_step / hevi_g_rk35_step */
int hevi_g_work_fields(const hevi_gplan *plan);
/* euler.nonlinear_rhs (euler.py:438-497) with DSS and no-flux projection */
int hevi_g_rhs(hevi_gplan *plan, const double *q, double *R, void *stream);
/* euler.vertical_restriction (euler.py:368-371) */
int hevi_g_linear_v(hevi_gplan *plan, const double *q, double *L, void *stream);
/* columnsolve.get_factors (factor_with_fallback): probe every column's
 * vertical lhs_schur on the device, banded LU (pivoted dense fallback) */
int hevi_g_factor(hevi_gplan *plan, double lam, int *nb_out, int *pivoted_out, void *stream);
/* the probed (unfactored) matrix of column `col` into A_host (M x M); col < 0: all (n_col x M x M) */
int hevi_g_column_matrix(hevi_gplan *plan, double lam, int col, double *A_host, void *stream);
/* ImplicitProblem.solve direct (imexcore.py:312-322 -> columnsolve.solve_direct) */
int hevi_g_solve(hevi_gplan *plan, double lam, const double *qe, double *q, void *stream);
/* imexcore.ark_imex_step, ARK2 1D-IMEX direct, Q in place; work: hevi_g_work_fields E-vectors */
int hevi_g_ark2_step(hevi_gplan *plan, double dt, const double *tab, double *Q, double *work, void *stream);
/* imexcore.rk35_step, Q in place */
int hevi_g_rk35_step(hevi_gplan *plan, double dt, double *Q, double *work, void *stream);
/* specgrid.apply_dss_many on nf fields (in may equal out) */
int hevi_g_dss(hevi_gplan *plan, const double *in, double *out, int nf, void *stream);
/* Discretization.gradc / grad_vc (vertical_only): out [3][nn]; divc / div_vc: in [3][nn], out [nn] */
int hevi_g_grad(hevi_gplan *plan, int vertical_only, const double *f, double *out, void *stream);
int hevi_g_div(hevi_gplan *plan, int vertical_only, const double *vec, double *out, void *stream);
int hevi_g_flags(hevi_gplan *plan, unsigned *flags, int reset, void *stream);
/* 3D-IMEX on the general mesh (ImplicitProblem dim "3d", or "1d" with
 * vertical_only): the Schur pieces of imexcore.py:200-298 on E-vectors,
 * euler.linear_operator (euler.py:313-365), and the Krylov solvers' plain
 * dot product over n doubles (krylov.py:46-55) */
int hevi_g_schur3_ua(hevi_gplan *plan, double lam, const double *qe, double *ua, double *Pe, void *stream);
int hevi_g_schur3_up(hevi_gplan *plan, double lam, int vertical_only, const double *P, double *up, void *stream);
int hevi_g_schur3_flux(hevi_gplan *plan, double lam, int vertical_only, const double *P, const double *vel,
                       double *out, void *stream);
int hevi_g_schur3_extract(hevi_gplan *plan, double lam, int vertical_only, const double *P, const double *ua,
                          const double *up, const double *qe, double *q, void *stream);
int hevi_g_linear3(hevi_gplan *plan, const double *q, double *out, void *stream);
int hevi_g_dot(hevi_gplan *plan, const double *x, const double *y, long long n, double *out_host, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* HEVI_H */
