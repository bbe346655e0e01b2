/*
 * mgpbd.h — C-ABI of libmgpbd.so, the B200-native (sm_100a) hot path of MGPBD (arXiv 2505.13390).
 *
 * One frame of PAPER.md Algorithm 1: predict, then n_iters outer iterations of
 * {evaluate C and grad C; re-assemble A = grad C M^-1 grad C^T + alpha_tilde into the fixed CSR
 * pattern; b = -C - alpha_tilde lambda (Eq. 3); lazily rebuild the
 * UA-AMG hierarchy; Galerkin A_{l+1} = P^T A_l P (Eq. 6,
 * PAPER.md:309); MGPCG with one V-cycle per iteration; dx = M^-1 grad C^T
 * dlambda (Eq. 5); lambda += dlambda; x += omega dx}, then v = (x - x_old)/dt.
 * Every step runs in this library's own CUDA kernels on the device; there is no CPU fallback.
 *
 * Conventions (all functions):
 *  - Ownership: input pointers are HOST memory borrowed for the duration of the call and copied.
 *    Output buffers are caller-owned host memory.  The context owns all device memory and frees it
 *    in mgpbd_destroy.
 *  - Errors: functions return an mgpbd_status and never throw across the ABI; the context keeps a
 *    last-error string (mgpbd_last_error).  Argument errors leave the state unchanged.  Solver
 *    errors (non-SPD coarsest matrix, non-finite values) are raised from device flags at the end
 *    of mgpbd_step; the state is then the completed (possibly polluted) frame.
 *  - Numbering: user numbering (constraint order and vertex order as passed to mgpbd_create) is
 *    preserved at the boundary; the level-l matrices returned by the test hooks are CSR with
 *    off-diagonals in ascending column order and the diagonal last in every row.
 *  - Threading: one context per host thread; all work is enqueued on cfg.stream (NULL = a stream
 *    the context creates) and every call returns after synchronising that stream.
 */
#ifndef MGPBD_H
#define MGPBD_H
#include <stdint.h>

#if defined(__GNUC__)
#define MGPBD_API __attribute__((visibility("default")))
#else
#define MGPBD_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mgpbd_ctx mgpbd_ctx; /* opaque; owns all device memory */

typedef enum {
    MGPBD_OK = 0,
    MGPBD_E_ARG = -1,        /* invalid argument (state unchanged) */
    MGPBD_E_CUDA = -2,       /* CUDA runtime error (message in mgpbd_last_error) */
    MGPBD_E_NCCL = -3,       /* multi-GPU communication error */
    MGPBD_E_OOM = -4,        /* device allocation failed */
    MGPBD_E_INDEFINITE = -5, /* the coarsest matrix of the hierarchy is not SPD (non-positive pivot in its
                                dense inversion).  A PCG iteration with <z,r> <= 0 (r != 0) is
                                NOT an error: it is counted in mgpbd_stats.indefinite_events, the frame
                                completes, and with cfg.resetup_on_indef the setup re-runs at the next frame */
    MGPBD_E_NONFINITE = -6,  /* NaN/Inf reached the right-hand side or the PCG scalars */
    MGPBD_E_STALL = -7       /* coarsening stalled with a coarsest level too large to invert */
} mgpbd_status;

typedef enum { MGPBD_DISTANCE = 2, MGPBD_TET_ARAP = 4 } mgpbd_kind; /* value = cardinality */

typedef struct {
    int32_t n_verts;
    const double* rest_pos; /* 3*n_verts, xyz interleaved (rest shape: L or D_m, V) */
    const double* pos;      /* 3*n_verts initial positions; NULL = rest_pos */
    const double* vel;      /* 3*n_verts initial velocities; NULL = 0 */
} mgpbd_mesh;

typedef struct {
    mgpbd_kind kind;        /* MGPBD_DISTANCE (cloth) or MGPBD_TET_ARAP (Eq. 8) */
    int32_t n_cons;         /* m = number of constraints = rows of A */
    const int32_t* verts;   /* kind*n_cons vertex ids, constraint-major */
} mgpbd_constraints;

typedef struct {
    int32_t precision;        /* 0: fp64 everywhere; 1: fp32 storage of A, h, P and level vectors
                                 with fp64 accumulation, fp64 setup, fp64 scalars and coarsest solve */
    double theta;             /* SOC threshold theta_s, 0.1 */
    int32_t k_nullspace;      /* near-kernel vectors per aggregate ("six distinct B"): 1 (default,
                                 reading c1) or 2..8 (k bootstrapped columns, per-aggregate
                                 thin QR, block coarse operators; one rank; readings c23-c25) */
    int32_t min_coarse;       /* coarsen while n_l >= min_coarse, 400 */
    int32_t max_levels;       /* 16 */
    double stall_ratio;       /* stop coarsening when n_{l+1}/n_l > stall_ratio, 0.9 */
    int32_t setup_interval;   /* lazy setup every k frames, 20 */
    int32_t bootstrap_sweeps; /* GS sweeps on A x = 0, 20 */
    int32_t power_iters;      /* power-method iterations for lambda_max(D^-1 A), 100 */
    double lambda_min_est;    /* user estimate of lambda_min, 0.1 */
    double lambda_safety;     /* omega = 2/(lambda_safety*lambda_max + lambda_min_est), 1.1: keeps the
                                 lazily-set omega below 2/lambda_max as A drifts (reading c9) */
    int32_t smoother_sweeps;  /* pre = post smoother steps, 2 (1..8) */
    int32_t pcg_iters;        /* MGPCG iterations per outer iteration (reading c10), 10 (<= 4090) */
    double omega_relax;       /* x += omega dx: 0.1 tets, 0.25 cloth */
    double gravity[3];        /* (0, -9.8, 0) */
    uint64_t seed;            /* hash seed (reading c0), 1 */
    int32_t device;           /* CUDA device ordinal */
    void* stream;             /* cudaStream_t, NULL = context-owned stream */
    int32_t max_dense_coarse; /* largest coarsest level inverted densely (default 2048; MGPBD_E_STALL above) */
    int32_t rank, world;      /* row partition of level 0 over `world` ranks, 0 <= rank < world */
    int32_t profile;          /* 1: record CUDA events around the level-0 matrix passes */
    const void* nccl_id;      /* world > 1: 128-byte ncclUniqueId shared by all ranks (mgpbd_nccl_unique_id on
                                 rank 0, broadcast by the caller); one process and one GPU per rank.  A non-NULL
                                 id with world == 1 runs the partitioned code path on one rank */
    void* vgroup;             /* alternative to nccl_id: a virtual-ranks group (mgpbd_vgroup_create) — `world`
                                 contexts in one process, one host thread each, all on one GPU (tests) */
    int32_t level0_operator;  /* hot level-0 matrix passes: 0 = stream the assembled CSR, 1 = matrix-free
                                 A x = H (H^T x) + at x from the scaled gradients (SURVEY.md §8(f) f4,
                                 PAPER.md:450); the CSR is assembled either way (Galerkin, diagonal).
                                 Default 1 */
    int32_t smoother;         /* V-cycle smoother: 0 = omega-Jacobi (default), 1 = Chebyshev
                                 (smoother_sweeps steps = polynomial degree; reading c20), 2 = multicolour
                                 Gauss-Seidel (forward pre / reversed post sweeps; reading c22; needs
                                 level0_operator = 0 and one rank) */
    double cheb_lower;        /* Chebyshev interval [cheb_lower * hi, hi] of D^-1 A, hi = lambda_safety *
                                 lambda_max (power method, lazily at setup: PAPER.md:320); 0.25 */
    int32_t backtrack;        /* 1: halve the relaxation omega (floor omega_min) whenever ||b|| of an outer
                                 iteration exceeds the previous one (reading c21); 0 */
    double omega_min;         /* 1e-3 */
    double residual_tol;      /* Alg. 1 l.12: stop the frame after the first outer iteration with
                                 ||b|| < residual_tol * ||b_0|| (one host read per iteration); 0 = off */
    double pcg_tol;           /* MGPCG convergence exit: the solve stops (remaining iterations become no-ops,
                                 decided on the device) at the first iteration k with ||r_k|| <= pcg_tol *
                                 ||b||; 0 = off: exactly pcg_iters iterations (reading c10) */
    double residual_abs;      /* Alg. 1 l.12 with an absolute eps ("||b|| < 1e-4"): stop the frame
                                 after the first outer iteration with ||b|| < residual_abs; 0 = off */
    int32_t resetup_on_indef; /* 1 (default): a frame in which a PCG iteration saw <z,r> <= 0 marks the
                                 hierarchy stale, so the setup re-runs at ite 0 of the next frame (reading
                                 c13 extension); 0: the literal lazy schedule of PAPER.md:215
                                 (setup only every setup_interval frames).  With lambda_safety = 1 this is
                                 the paper's literal mode */
    int32_t omega_refresh_iters; /* 0 (default): the smoother weights are fixed at setup (lazy).
                                 > 0: at ite 0 of every frame WITHOUT a setup, this many further power
                                 iterations per level on the current fp64 level matrices, started from the
                                 iterate the previous setup / refresh left, re-derive lambda_max and the
                                 smoother coefficients (reading c26).
                                 Costs the fp64 Galerkin refresh + the iterations + one graph re-capture
                                 per frame */
    double time_budget_ms;    /* Alg. 1 l.12 "timeBudgetExhausted": stop the frame after the first
                                 outer iteration that completes more than this many ms (device time, CUDA events)
                                 after the frame started (one host synchronisation per outer iteration); 0 = off.
                                 Machine-dependent by definition (reading c21) */
} mgpbd_config;

#define MGPBD_MAX_LEVELS 16
#define MGPBD_MAX_ITERS 256            /* outer iterations recorded in mgpbd_stats.b_norm */
#define MGPBD_MAX_FRAME_ITERS 1000000  /* outer iterations per frame ("maxiter (1e5)") */

typedef struct {
    int32_t n_levels;
    int64_t n[MGPBD_MAX_LEVELS], nnz[MGPBD_MAX_LEVELS];
    double op_complexity;              /* sum nnz_l / nnz_0 (Table 1 "C") */
    double omega[MGPBD_MAX_LEVELS];    /* omega-Jacobi weight per level (coarsest: 0) */
    int32_t n_colours;                 /* colours of the level-0 GS bootstrap */
    int32_t setup_ran;                 /* setup ran in the last frame */
    int32_t n_b;                       /* outer iterations recorded in b_norm */
    double b_norm[MGPBD_MAX_ITERS];    /* ||b||_2 per outer iteration of the last frame (the first
                                          MGPBD_MAX_ITERS; n_b counts them, b_last is the final one) */
    int64_t frame;                     /* frames stepped so far */
    /* profile == 1 only: summed CUDA-event time of the level-0 matrix-pass kernels (smoother
       sweeps, residual, PCG SpMV) in the last frame, their launch count and algorithmic bytes */
    double l0_pass_ms;
    int64_t l0_pass_launches;
    double l0_pass_bytes;
    double ms_setup;                   /* CUDA-event time of the setup in the last frame */
    double ms_frame;                   /* CUDA-event time of the last frame */
    int64_t kernel_launches;           /* this library's kernel launches in the last frame */
    int32_t indefinite_events;         /* PCG iterations of the last frame with <z,r> <= 0 (r != 0):
                                          the lazily-set omega went stale; setup re-runs next frame */
    int32_t rank, world;               /* partitioned run: this rank / number of ranks (1 otherwise) */
    int32_t row_begin, row_end;        /* level-0 rows this rank owns */
    int64_t halo_rows;                 /* level-0 x entries received per halo exchange */
    double omega_relax;                /* relaxation omega at the end of the last frame (backtracking) */
    /* phase times of the last frame in ms (recorded only with profile = 1, i.e. eager launches; else 0):
       constraint evaluation + assembly / matrix-free refresh, Galerkin refresh + coarsest inverse,
       V-cycles, the rest of MGPCG, position / lambda update */
    double ms_assemble, ms_galerkin, ms_vcycle, ms_pcg_other, ms_update;
    int32_t iters_run;                 /* outer iterations the last frame ran (< n_iters after an l.12 exit) */
    double b_last;                     /* ||b||_2 of its last outer iteration */
} mgpbd_stats;

/* Fill *cfg with the defaults listed above.  Never fails for a non-NULL cfg. */
MGPBD_API mgpbd_status mgpbd_config_default(mgpbd_config* cfg);

/* Create a context: validates inputs, uploads them, computes rest data (L, or D_m^-1 and V) and the
 * fixed CSR pattern of A ((i,j) stored iff constraints i, j share a vertex; sorted
 * off-diagonals, diagonal last) on the device.  inv_mass: n_verts inverse masses, 0 = pinned.
 * compliance: per-constraint alpha (NOT divided by dt^2; alpha_tilde = alpha/dt^2 per step).
 * Errors: MGPBD_E_ARG (NULL pointers, vertex ids out of range, repeated vertex in a constraint,
 * negative mass/compliance, degenerate rest tet, bad config), MGPBD_E_CUDA/OOM. */
MGPBD_API mgpbd_status mgpbd_create(const mgpbd_mesh* mesh, const mgpbd_constraints* cons,
                          const double* inv_mass, const double* compliance,
                          const mgpbd_config* cfg, mgpbd_ctx** out);

/* Mark the hierarchy stale: it is rebuilt at ite 0 of the next mgpbd_step (Alg. 1 l.7). */
MGPBD_API mgpbd_status mgpbd_setup_hierarchy(mgpbd_ctx* ctx);

/* One frame of Algorithm 1 with n_iters outer iterations (1..MGPBD_MAX_FRAME_ITERS) and time step dt > 0.
 * Setup runs at ite 0 when frame % setup_interval == 0 or the hierarchy is stale.  Synchronises at
 * the end and checks the device flags: MGPBD_E_NONFINITE (NaN/Inf PCG scalar), MGPBD_E_INDEFINITE
 * (non-SPD coarsest matrix).  <z,r> <= 0 in PCG is counted (mgpbd_stats.indefinite_events), not
 * returned. */
MGPBD_API mgpbd_status mgpbd_step(mgpbd_ctx* ctx, double dt, int32_t n_iters);

/* CUDA-event timing of the level-0 matrix passes (mgpbd_stats.l0_pass_*): 0 off; 1 eager — the
 * per-iteration CUDA graphs are not used, the same kernels launch eagerly between event records (and the
 * phase times ms_* are recorded); 2 in-graph — the pass events are captured as nodes of the replayed
 * per-iteration graph (the launch configuration the bench times); each replay overwrites them, so the last
 * replay's pass durations stand for every outer iteration.  Errors: MGPBD_E_ARG for a NULL context. */
MGPBD_API mgpbd_status mgpbd_set_profiling(mgpbd_ctx* ctx, int32_t on);

/* Upload a new state (3*n_verts each; vel may be NULL = unchanged). */
MGPBD_API mgpbd_status mgpbd_set_state(mgpbd_ctx* ctx, const double* pos, const double* vel);

/* Read back positions / velocities (3*n_verts doubles) and lambda (n_cons doubles, user order). */
MGPBD_API mgpbd_status mgpbd_get_positions(mgpbd_ctx* ctx, double* out);
MGPBD_API mgpbd_status mgpbd_get_velocities(mgpbd_ctx* ctx, double* out);
MGPBD_API mgpbd_status mgpbd_get_lambda(mgpbd_ctx* ctx, double* out);
MGPBD_API mgpbd_status mgpbd_get_stats(mgpbd_ctx* ctx, mgpbd_stats* out);

/* ---- test hooks (hierarchy as built by the last setup; level l in user numbering) ---- */
MGPBD_API mgpbd_status mgpbd_get_level_sizes(mgpbd_ctx* ctx, int32_t l, int64_t* n, int64_t* nnz);
/* CSR of level l (rowptr n+1, cols nnz, vals nnz as fp64): current values of the hot loop. */
MGPBD_API mgpbd_status mgpbd_get_level(mgpbd_ctx* ctx, int32_t l, int64_t* rowptr, int32_t* cols, double* vals);
/* Level-l prolongator values P_i (n_l doubles, one per row; column = aggregate of row i); k_nullspace = 1
 * only (MGPBD_E_ARG otherwise: use mgpbd_get_prolongator_csr). */
MGPBD_API mgpbd_status mgpbd_get_prolongator(mgpbd_ctx* ctx, int32_t l, double* p_vals);
/* Level-l prolongator as CSR (n_l x n_{l+1}, columns ascending per row): *nnz always; rowptr (n_l + 1),
 * col and val (nnz each) when non-NULL.  k_nullspace = 1: one entry per row, column = aggregate, value =
 * P_i; k > 1 (readings c24/c25): row i holds the r_a (<= k) entries of its aggregate's
 * thin-QR factor Q_a in columns off_a .. off_a + r_a - 1. */
MGPBD_API mgpbd_status mgpbd_get_prolongator_csr(mgpbd_ctx* ctx, int32_t l, int64_t* nnz, int64_t* rowptr,
                                                 int32_t* col, double* val);
/* Level-l aggregate index per node (n_l int32). */
MGPBD_API mgpbd_status mgpbd_get_aggregates(mgpbd_ctx* ctx, int32_t l, int32_t* out);
/* Level-0 near-kernel vector(s) B after the GS bootstrap: n_0 x k_nullspace doubles, column-major (column c
 * starts at out + c n_0; reading c23). */
MGPBD_API mgpbd_status mgpbd_get_near_kernel(mgpbd_ctx* ctx, double* out);
/* Run the setup on caller-given level-0 values (nnz doubles in the pattern's CSR order), then the
 * Galerkin refresh and coarse inversion on the same values (identical-input-bits tests). */
MGPBD_API mgpbd_status mgpbd_debug_setup_from(mgpbd_ctx* ctx, const double* A0_values);
/* Apply one V-cycle / K MGPCG iterations of the current hierarchy to host b (n_0) -> host x. */
MGPBD_API mgpbd_status mgpbd_debug_vcycle(mgpbd_ctx* ctx, const double* b, double* x);
MGPBD_API mgpbd_status mgpbd_debug_pcg(mgpbd_ctx* ctx, const double* b, int32_t iters, double* x);
/* Alg. 1 l.1-7 of the next frame without the solve: predict (positions become the
 * predicted x~, velocities get dt g), lambda = 0, evaluate the constraints and refresh the hot level-0
 * operator at x~ (matrix-free when configured), run the setup if one is due (frame % setup_interval
 * == 0 or stale), then the Galerkin refresh and coarsest inverse — so debug_vcycle / debug_pcg apply
 * exactly the operators mgpbd_step's first outer iteration uses.  The frame counter is not advanced.
 * Errors: MGPBD_E_ARG for dt <= 0. */
MGPBD_API mgpbd_status mgpbd_debug_prepare(mgpbd_ctx* ctx, double dt);
/* Measurement hook: `reps` (1..4096) level-0 SpMV+dot passes of the hot operator on the current state,
 * captured as one CUDA graph and timed with events around its replay (no launch gaps).  *ms = device
 * time, *bytes = the passes' algorithmic bytes.  Needs a stepped context and one rank; E_ARG otherwise. */
MGPBD_API mgpbd_status mgpbd_pass_burst(mgpbd_ctx* ctx, int32_t reps, double* ms, double* bytes);

/* ---- multi-GPU (row-partitioned level 0; coarse levels and setup replicated) ----
 * Every rank calls every function with the same inputs.  Per level-0 matrix pass the rank exchanges
 * the halo of x with the ranks owning the rows its rows reference; dots, the level-1 restriction, the
 * level-1 Galerkin values and dlambda are summed over ranks.  get_positions/get_lambda return the
 * global arrays on every rank; get_level(0) values are current only for the rank's own rows. */
/* Write a fresh 128-byte NCCL unique id (host call; rank 0 creates it, the caller broadcasts it). */
MGPBD_API mgpbd_status mgpbd_nccl_unique_id(void* out128);
/* Virtual ranks: a group for `world` contexts created in one process (one host thread per context). */
MGPBD_API mgpbd_status mgpbd_vgroup_create(int32_t world, void** out);
MGPBD_API void mgpbd_vgroup_destroy(void* group);
/* Host-only partition logic (no device work): bounds[world+1] = row blocks balanced by nonzeros. */
MGPBD_API mgpbd_status mgpbd_partition_rows(const int64_t* rowptr, int32_t n, int32_t world, int32_t* bounds);
/* Host-only halo plan: recv[(q*world+p)*2 + {0,1}] = [a, b) rows rank q receives from rank p, given each
 * rank's referenced column window [minc[q], maxc[q]]. */
MGPBD_API mgpbd_status mgpbd_halo_plan(const int32_t* bounds, const int32_t* minc, const int32_t* maxc,
                                       int32_t world, int32_t* recv);

MGPBD_API const char* mgpbd_last_error(const mgpbd_ctx* ctx);
MGPBD_API void mgpbd_destroy(mgpbd_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* MGPBD_H */
