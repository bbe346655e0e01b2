/*
 * MGPBD ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, serial fp64 CPU implementation of one MGPBD frame (Algorithm 1,
 * PAPER.md:203-227) and of every step on its hot path.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  It shares no code,
 * header, table or constant generator with the CUDA library (paper_2505_13390_b200/csrc).
 *
 * Every function cites the passage it follows (PAPER.md line; SURVEY.md §8(c) reading id).
 * Parity status per function is listed in DESIGN.md §"Oracle pins".  "parity unpinned":
 * the *partition* produced by orc_aggregate is unpinned w.r.t. the paper (its visiting order
 * is unstated; reading c2) — its invariants are pinned by tests.
 */
#ifndef MGPBD_ORACLE_H
#define MGPBD_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    double theta;            /* SOC threshold, PAPER.md:250 (0.1) */
    int32_t min_coarse;      /* coarsen while n >= this, PAPER.md:241 (400) */
    int32_t max_levels;      /* 16 (reading c7) */
    double stall_ratio;      /* 0.9 (reading c7) */
    int32_t setup_interval;  /* 20 */
    int32_t bootstrap_sweeps;/* 20 */
    int32_t power_iters;     /* 100 (reading c9) */
    double lambda_min_est;   /* 0.1 */
    double lambda_safety;    /* omega = 2/(safety*lambda_max + lambda_min_est); 1.1 (reading c9) */
    int32_t smoother_sweeps; /* 2 */
    int32_t pcg_iters;       /* 10 (reading c10) */
    double omega_relax;      /* 0.1 tet / 0.25 cloth */
    double gravity[3];       /* (0,-9.8,0) */
    uint64_t seed;           /* 1 */
    int32_t smoother;        /* 0 omega-Jacobi, 1 Chebyshev (c20), 2 multicolour GS (c22) */
    double cheb_lower;       /* Chebyshev interval [cheb_lower*hi, hi], hi = safety*lambda_max; 0.25 (c20) */
    int32_t backtrack;       /* 1: halve omega when ||b|| rises (reading c21); 0 */
    double omega_min;        /* floor of the halving; 1e-3 */
    double residual_tol;     /* Alg. 1 l.12: break once ||b|| < residual_tol * ||b_0||; 0 = off (c11/c21) */
    double pcg_tol;          /* MGPCG stops once ||r_k|| <= pcg_tol ||b||; 0 = off, fixed pcg_iters (c10) */
    int32_t resetup_on_indef;/* 1: a frame with a PCG iteration <z,r> <= 0 marks the hierarchy stale, so setup
                                re-runs at ite 0 of the next frame (reading c13 extension); 0: the literal
                                schedule of PAPER.md:215 (setup only every setup_interval frames).  Default 1 */
    double residual_abs;     /* Alg. 1 l.12 absolute eps ("||b|| < 1e-4"): break once ||b|| < it; 0 = off */
    int32_t omega_refresh_iters; /* > 0: at ite 0 of frames without a setup, omega_l / the Chebyshev interval are
                                    re-estimated by this many power iterations on the current level matrices from
                                    the last normalised iterate (reading c26); 0 = omega only at setup */
    int32_t k_nullspace;     /* near-kernel vectors per aggregate ("six distinct B"; reading c1):
                                1 (default) or up to 6 */
    double time_budget_ms;   /* Alg. 1 l.12 "timeBudgetExhausted": break after the first outer iteration
                                that ends more than this many ms (wall clock) after the frame started; 0 = off.
                                Machine-dependent by definition (reading c21) */
} orc_config;

void orc_config_default(orc_config* c);

/* ---- hash (reading c0) ---- */
uint64_t orc_mix64(uint64_t z);
uint64_t orc_key(uint64_t seed, int stream, int level, uint64_t i);
double orc_uniform(uint64_t seed, int stream, int level, uint64_t i);

/* ---- constraints (a1) ---- */
void orc_rest_distance(int32_t m, const int32_t* verts, const double* X, double* rest_len);
int orc_rest_arap(int32_t m, const int32_t* verts, const double* X, double* Dm_inv, double* vol);
void orc_eval_distance(int32_t m, const int32_t* verts, const double* x, const double* rest_len,
                       double* C, double* g /* m*2*3 */);
void orc_polar(const double* F /*9 row-major*/, double* R /*9*/);
void orc_eval_arap(int32_t m, const int32_t* verts, const double* x, const double* Dm_inv,
                   double* C, double* g /* m*4*3 */);

/* ---- pattern + assembly (a2) ---- */
int64_t orc_pattern(int32_t m, int kind, const int32_t* verts, int32_t n_verts,
                    int64_t* rowptr /* m+1 or NULL */, int32_t* col /* nnz or NULL */);
void orc_assemble(int32_t m, int kind, const int32_t* verts, const double* w, const double* g,
                  const double* alpha_tilde, const int64_t* rowptr, const int32_t* col, double* val);
void orc_assemble_rows(int32_t nrows, const int32_t* rows, int kind, const int32_t* verts, const double* w,
                       const double* g, const double* alpha_tilde, const int64_t* rowptr, const int32_t* col,
                       double* val);
void orc_rhs(int32_t m, const double* C, const double* alpha_tilde, const double* lambda, double* b);
void orc_apply_dx(int32_t m, int kind, const int32_t* verts, int32_t n_verts, const double* w,
                  const double* g, const double* dlambda, double* dx /* 3*n_verts */);

/* ---- sparse helpers ---- */
void orc_spmv(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val,
              const double* x, double* y);

/* ---- setup (a3-a8) ---- */
void orc_soc(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val, double theta,
             uint8_t* strong);
int32_t orc_aggregate(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val,
                      const uint8_t* strong, uint64_t seed, int level, int32_t* agg);
int32_t orc_colour(int32_t n, const int64_t* rowptr, const int32_t* col, uint64_t seed,
                   int32_t* colour);
void orc_gs_bootstrap(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val,
                      const int32_t* colour, int32_t sweeps, uint64_t seed, double* B);
void orc_prolongator(int32_t n, const int32_t* agg, int32_t n_agg, const double* B, double* P,
                     double* B_next);
int64_t orc_galerkin(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val,
                     const int32_t* agg, const double* P, int32_t n_agg,
                     int64_t* crowptr, int32_t* ccol, double* cval /* all NULL => count only */);
/* k > 1 near kernel (f2; readings c23-c25): k bootstrapped columns (column-major n x k), per-aggregate
 * MGS thin QR injection into a CSR prolongator, general Galerkin P^T A P. */
void orc_gs_bootstrap_k(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val,
                        const int32_t* colour, int32_t sweeps, uint64_t seed, int32_t k, double* B);
int32_t orc_prolongator_qr(int32_t n, const int32_t* agg, int32_t n_agg, int32_t k, const double* B,
                           double rank_tol, int32_t* coff, int64_t* pptr, int32_t* pcol, double* pval,
                           double* B_next, int32_t ld_next);
int64_t orc_galerkin_p(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val,
                       const int64_t* pptr, const int32_t* pcol, const double* pval, int32_t nc,
                       int64_t* crowptr, int32_t* ccol, double* cval);
double orc_power_from(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val, int32_t iters,
                      double* v /* normalised start, in/out */);
double orc_power(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val,
                 int32_t iters, uint64_t seed, int level);
int orc_cholesky(int32_t n, const double* A /* dense n*n */, double* L /* n*n */);
void orc_chol_solve(int32_t n, const double* L, const double* b, double* x);

/* ---- hierarchy / solve (a6-a11) ---- */
typedef struct orc_hier orc_hier;
orc_hier* orc_hier_build(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val,
                         const orc_config* cfg);
int orc_hier_refresh(orc_hier* h, const double* val0); /* new A_0 values: Galerkin + coarse factor */
void orc_hier_refresh_omega(orc_hier* h, int32_t iters);   /* reading c26: per-frame omega refresh */
void orc_hier_free(orc_hier* h);
int orc_hier_levels(const orc_hier* h);
void orc_hier_level_size(const orc_hier* h, int l, int32_t* n, int64_t* nnz);
void orc_hier_get_level(const orc_hier* h, int l, int64_t* rowptr, int32_t* col, double* val);
void orc_hier_get_agg(const orc_hier* h, int l, int32_t* agg);
void orc_hier_get_P(const orc_hier* h, int l, double* P);
double orc_hier_omega(const orc_hier* h, int l);
/* Chebyshev interval centre theta and half-width delta of level l (reading c20) */
void orc_hier_cheb(const orc_hier* h, int l, double* theta, double* delta);
/* one smoothing pass (the level's configured smoother, cfg.smoother_sweeps steps) on A x = b;
 * post = 1: the post-smoother (GS: reversed colour order) */
void orc_hier_smooth(const orc_hier* h, int l, const double* b, double* x, int post);
void orc_hier_get_B0(const orc_hier* h, double* B);   /* n_0 x k, column-major */
void orc_hier_get_P_csr(const orc_hier* h, int l, int64_t* nnz, int64_t* rowptr, int32_t* col, double* val);
int32_t orc_hier_n_colours(const orc_hier* h);
void orc_vcycle(const orc_hier* h, const double* b, double* x);
int orc_pcg(const orc_hier* h, const double* b, int32_t iters, double* x, double* rz_trace);

/* ---- simulation (Algorithm 1) ---- */
typedef struct orc_sim orc_sim;
orc_sim* orc_sim_create(int kind, int32_t n_verts, int32_t m, const int32_t* verts,
                        const double* rest_pos, const double* pos, const double* vel,
                        const double* inv_mass, const double* compliance, const orc_config* cfg);
int orc_sim_step(orc_sim* s, double dt, int32_t n_iters);
void orc_sim_mark_stale(orc_sim* s);
int32_t orc_sim_indefinite_events(const orc_sim* s);
int32_t orc_sim_setups(const orc_sim* s);          /* setups run since creation (Alg. 1 l.7) */
double orc_sim_setup_ms(const orc_sim* s);         /* wall time of the last frame's setup (0 if none) */
void orc_sim_get(const orc_sim* s, double* x, double* v, double* lambda);
void orc_sim_set(orc_sim* s, const double* x, const double* v);
const orc_hier* orc_sim_hier(const orc_sim* s);
int64_t orc_sim_nnz(const orc_sim* s);
void orc_sim_get_A(const orc_sim* s, int64_t* rowptr, int32_t* col, double* val);
void orc_sim_get_b_norms(const orc_sim* s, double* out, int32_t n);
int32_t orc_sim_iters_used(const orc_sim* s);      /* outer iterations run by the last frame */
double orc_sim_omega(const orc_sim* s);            /* relaxation omega at the end of the last frame */
void orc_sim_free(orc_sim* s);

#ifdef __cplusplus
}
#endif
#endif
