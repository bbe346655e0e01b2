/*
 * MGPBD ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Plain serial fp64 C, compiled with -O2 -ffp-contract=off, no fast-math.  Each function
 * follows the paper's definition or algorithm step by step; where the paper is silent the
 * SURVEY.md §8(c) reading (c0..c19, restated in DESIGN.md) is cited.
 */
#define _POSIX_C_SOURCE 199309L
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define OMAX(a, b) ((a) > (b) ? (a) : (b))
#define ORC_RANK_TOL 1e-10  /* QR column drop threshold, relative to the column norm (reading c24) */

static void* xmalloc(size_t n) { void* p = malloc(n ? n : 1); if (!p) abort(); return p; }
static void* xcalloc(size_t n, size_t s) { void* p = calloc(n ? n : 1, s ? s : 1); if (!p) abort(); return p; }

void orc_config_default(orc_config* c) {
    c->theta = 0.1; c->min_coarse = 400; c->max_levels = 16; c->stall_ratio = 0.9;
    c->setup_interval = 20; c->bootstrap_sweeps = 20; c->power_iters = 100;
    c->lambda_min_est = 0.1; c->lambda_safety = 1.1; c->smoother_sweeps = 2; c->pcg_iters = 10; c->omega_relax = 0.1;
    c->smoother = 0; c->cheb_lower = 0.25;
    c->backtrack = 0; c->omega_min = 1e-3; c->residual_tol = 0.0; c->pcg_tol = 0.0;
    c->resetup_on_indef = 1; c->residual_abs = 0.0; c->k_nullspace = 1; c->omega_refresh_iters = 0;
    c->time_budget_ms = 0.0;
    c->gravity[0] = 0.0; c->gravity[1] = -9.8; c->gravity[2] = 0.0; c->seed = 1;
}

/* ------------------------------------------------------------------------------------------
 * Hash, reading c0 ("selecting a node", "randomly sampled").
 * mix64 is the splitmix64 finaliser; key(stream,l,i) = mix64(mix64(seed^(stream<<56)^(l<<48))^i)
 * and U = ((key>>11)+0.5)*2^-53 in (0,1).
 * ------------------------------------------------------------------------------------------ */
uint64_t orc_mix64(uint64_t z) {
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27; z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}
uint64_t orc_key(uint64_t seed, int stream, int level, uint64_t i) {
    uint64_t base = seed ^ ((uint64_t)stream << 56) ^ ((uint64_t)level << 48);
    return orc_mix64(orc_mix64(base) ^ i);
}
double orc_uniform(uint64_t seed, int stream, int level, uint64_t i) {
    return ((double)(orc_key(seed, stream, level, i) >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}

/* ------------------------------------------------------------------------------------------
 * Constraints (a1).
 * ------------------------------------------------------------------------------------------ */

/* Distance rest length L = |X_a - X_b| (PAPER.md:441 cloth "distance constraints"; c16). */
void orc_rest_distance(int32_t m, const int32_t* verts, const double* X, double* rest_len) {
    for (int32_t j = 0; j < m; ++j) {
        const double* a = X + 3 * (int64_t)verts[2 * j];
        const double* b = X + 3 * (int64_t)verts[2 * j + 1];
        double d0 = a[0] - b[0], d1 = a[1] - b[1], d2 = a[2] - b[2];
        rest_len[j] = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
    }
}

static double det3(const double* M) {
    return M[0] * (M[4] * M[8] - M[5] * M[7]) - M[1] * (M[3] * M[8] - M[5] * M[6]) +
           M[2] * (M[3] * M[7] - M[4] * M[6]);
}

/* Rest shape D_m (columns X_k - X_0, k=1..3), its inverse, and V = |det D_m|/6. */
int orc_rest_arap(int32_t m, const int32_t* verts, const double* X, double* Dm_inv, double* vol) {
    int bad = 0;
    for (int32_t j = 0; j < m; ++j) {
        const double* x0 = X + 3 * (int64_t)verts[4 * j];
        double D[9];
        for (int c = 0; c < 3; ++c) {
            const double* xc = X + 3 * (int64_t)verts[4 * j + 1 + c];
            for (int r = 0; r < 3; ++r) D[r * 3 + c] = xc[r] - x0[r];
        }
        double det = det3(D);
        double* Di = Dm_inv + 9 * (int64_t)j;
        vol[j] = fabs(det) / 6.0;
        if (det == 0.0) { memset(Di, 0, 9 * sizeof(double)); bad = 1; continue; }
        /* inverse = adjugate / det */
        Di[0] = (D[4] * D[8] - D[5] * D[7]) / det;
        Di[1] = (D[2] * D[7] - D[1] * D[8]) / det;
        Di[2] = (D[1] * D[5] - D[2] * D[4]) / det;
        Di[3] = (D[5] * D[6] - D[3] * D[8]) / det;
        Di[4] = (D[0] * D[8] - D[2] * D[6]) / det;
        Di[5] = (D[2] * D[3] - D[0] * D[5]) / det;
        Di[6] = (D[3] * D[7] - D[4] * D[6]) / det;
        Di[7] = (D[1] * D[6] - D[0] * D[7]) / det;
        Di[8] = (D[0] * D[4] - D[1] * D[3]) / det;
    }
    return bad;
}

/* Distance constraint C = |x_a - x_b| - L; grad_a = u, grad_b = -u; |d| <= 1e-12 => zero
 * gradients (reading c16). */
void orc_eval_distance(int32_t m, const int32_t* verts, const double* x, const double* rest_len,
                       double* C, double* g) {
    for (int32_t j = 0; j < m; ++j) {
        const double* a = x + 3 * (int64_t)verts[2 * j];
        const double* b = x + 3 * (int64_t)verts[2 * j + 1];
        double d[3] = {a[0] - b[0], a[1] - b[1], a[2] - b[2]};
        double len = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        C[j] = len - rest_len[j];
        double* gj = g + 6 * (int64_t)j;
        for (int r = 0; r < 3; ++r) {
            double u = len > 1e-12 ? d[r] / len : 0.0;
            gj[r] = u;
            gj[3 + r] = -u;
        }
    }
}

/* Polar rotation R of F ("R is the rotation matrix decomposed from F"):
 * F = U S V^T by one-sided (Hestenes) Jacobi; R = U V^T; if det R < 0 the column of U of the
 * smallest singular value is negated; F = 0 => R = I (reading c15). */
void orc_polar(const double* F, double* R) {
    double A[9], V[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    int allzero = 1;
    for (int k = 0; k < 9; ++k) { A[k] = F[k]; if (F[k] != 0.0) allzero = 0; }
    if (allzero) { memcpy(R, V, sizeof V); return; }
    static const int PQ[3][2] = {{0, 1}, {0, 2}, {1, 2}};
    for (int sweep = 0; sweep < 60; ++sweep) {
        int rotated = 0;
        for (int t = 0; t < 3; ++t) {
            int p = PQ[t][0], q = PQ[t][1];
            double al = 0, be = 0, ga = 0;
            for (int r = 0; r < 3; ++r) {
                al += A[r * 3 + p] * A[r * 3 + p];
                be += A[r * 3 + q] * A[r * 3 + q];
                ga += A[r * 3 + p] * A[r * 3 + q];
            }
            if (ga == 0.0 || fabs(ga) <= 1e-15 * sqrt(al * be)) continue;
            rotated = 1;
            double zeta = (be - al) / (2.0 * ga);
            double t_ = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            double c = 1.0 / sqrt(1.0 + t_ * t_), s = c * t_;
            for (int r = 0; r < 3; ++r) {
                double ap = A[r * 3 + p], aq = A[r * 3 + q];
                A[r * 3 + p] = c * ap - s * aq;
                A[r * 3 + q] = s * ap + c * aq;
                double vp = V[r * 3 + p], vq = V[r * 3 + q];
                V[r * 3 + p] = c * vp - s * vq;
                V[r * 3 + q] = s * vp + c * vq;
            }
        }
        if (!rotated) break;
    }
    /* singular values = column norms; order descending */
    double sg[3];
    int ord[3] = {0, 1, 2};
    for (int k = 0; k < 3; ++k)
        sg[k] = sqrt(A[k] * A[k] + A[3 + k] * A[3 + k] + A[6 + k] * A[6 + k]);
    for (int a = 0; a < 3; ++a)
        for (int b = a + 1; b < 3; ++b)
            if (sg[ord[b]] > sg[ord[a]]) { int t = ord[a]; ord[a] = ord[b]; ord[b] = t; }
    double U[9], Vs[9];
    double smax = sg[ord[0]];
    int rank = 0;
    for (int k = 0; k < 3; ++k) {
        int c = ord[k];
        for (int r = 0; r < 3; ++r) Vs[r * 3 + k] = V[r * 3 + c];
        if (sg[c] > 1e-14 * smax) {
            for (int r = 0; r < 3; ++r) U[r * 3 + k] = A[r * 3 + c] / sg[c];
            rank = k + 1;
        }
    }
    if (rank < 2) { /* complete U's second column orthogonal to the first */
        double u0[3] = {U[0], U[3], U[6]};
        double e[3] = {0, 0, 0};
        int ax = (fabs(u0[0]) <= fabs(u0[1]) && fabs(u0[0]) <= fabs(u0[2])) ? 0 : (fabs(u0[1]) <= fabs(u0[2]) ? 1 : 2);
        e[ax] = 1.0;
        double c1[3] = {u0[1] * e[2] - u0[2] * e[1], u0[2] * e[0] - u0[0] * e[2], u0[0] * e[1] - u0[1] * e[0]};
        double nn = sqrt(c1[0] * c1[0] + c1[1] * c1[1] + c1[2] * c1[2]);
        for (int r = 0; r < 3; ++r) U[r * 3 + 1] = c1[r] / nn;
    }
    if (rank < 3) { /* third column = u0 x u1 */
        double u0[3] = {U[0], U[3], U[6]}, u1[3] = {U[1], U[4], U[7]};
        U[2] = u0[1] * u1[2] - u0[2] * u1[1];
        U[5] = u0[2] * u1[0] - u0[0] * u1[2];
        U[8] = u0[0] * u1[1] - u0[1] * u1[0];
    }
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
            R[r * 3 + c] = U[r * 3] * Vs[c * 3] + U[r * 3 + 1] * Vs[c * 3 + 1] + U[r * 3 + 2] * Vs[c * 3 + 2];
    if (det3(R) < 0.0) {
        for (int r = 0; r < 3; ++r) U[r * 3 + 2] = -U[r * 3 + 2];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c)
                R[r * 3 + c] = U[r * 3] * Vs[c * 3] + U[r * 3 + 1] * Vs[c * 3 + 1] + U[r * 3 + 2] * Vs[c * 3 + 2];
    }
}

/* ARAP constraint, Eq. 8: C = ||F - R||_F^2 with F = D_s D_m^{-1} (literal squared
 * form, reading c15); dC/dF = 2(F - R); G = 2(F - R) D_m^{-T}; g_{1..3} = columns of G;
 * g_0 = -(g_1+g_2+g_3).  Non-finite F => C = 0, g = 0. */
void orc_eval_arap(int32_t m, const int32_t* verts, const double* x, const double* Dm_inv,
                   double* C, double* g) {
    for (int32_t j = 0; j < m; ++j) {
        const int32_t* tv = verts + 4 * (int64_t)j;
        const double* x0 = x + 3 * (int64_t)tv[0];
        double Ds[9];
        for (int c = 0; c < 3; ++c) {
            const double* xc = x + 3 * (int64_t)tv[1 + c];
            for (int r = 0; r < 3; ++r) Ds[r * 3 + c] = xc[r] - x0[r];
        }
        const double* Di = Dm_inv + 9 * (int64_t)j;
        double F[9];
        int finite = 1;
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) {
                double s = 0;
                for (int k = 0; k < 3; ++k) s += Ds[r * 3 + k] * Di[k * 3 + c];
                F[r * 3 + c] = s;
                if (!isfinite(s)) finite = 0;
            }
        double* gj = g + 12 * (int64_t)j;
        if (!finite) { C[j] = 0.0; memset(gj, 0, 12 * sizeof(double)); continue; }
        double R[9], E[9];
        orc_polar(F, R);
        double c2 = 0;
        for (int k = 0; k < 9; ++k) { E[k] = F[k] - R[k]; c2 += E[k] * E[k]; }
        C[j] = c2;
        for (int r = 0; r < 3; ++r) gj[r] = 0.0;
        for (int c = 0; c < 3; ++c)
            for (int r = 0; r < 3; ++r) {
                double s = 0;
                for (int k = 0; k < 3; ++k) s += E[r * 3 + k] * Di[c * 3 + k];
                gj[3 * (1 + c) + r] = 2.0 * s;
            }
        for (int r = 0; r < 3; ++r) gj[r] = -(gj[3 + r] + gj[6 + r] + gj[9 + r]);
    }
}

/* ------------------------------------------------------------------------------------------
 * Pattern and assembly (a2): "stored in CSR format with three fixed length
 * arrays. For each row, we store the off-diagonal terms first and put the diagonal terms at
 * last."  (i,j) stored iff constraints i and j share a vertex.
 * ------------------------------------------------------------------------------------------ */
static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

/* vertex -> incident constraints, constraints ascending */
static void incidence(int32_t m, int kind, const int32_t* verts, int32_t nv, int64_t** pptr, int32_t** plist) {
    int64_t* ptr = xcalloc((size_t)nv + 1, sizeof(int64_t));
    for (int64_t e = 0; e < (int64_t)m * kind; ++e) ptr[verts[e] + 1]++;
    for (int32_t v = 0; v < nv; ++v) ptr[v + 1] += ptr[v];
    int32_t* list = xmalloc(sizeof(int32_t) * (size_t)m * kind);
    int64_t* fill = xmalloc(sizeof(int64_t) * ((size_t)nv + 1));
    memcpy(fill, ptr, sizeof(int64_t) * ((size_t)nv + 1));
    for (int32_t j = 0; j < m; ++j)
        for (int k = 0; k < kind; ++k) list[fill[verts[(int64_t)j * kind + k]]++] = j;
    free(fill);
    *pptr = ptr; *plist = list;
}

int64_t orc_pattern(int32_t m, int kind, const int32_t* verts, int32_t n_verts, int64_t* rowptr, int32_t* col) {
    int64_t* iptr; int32_t* ilist;
    incidence(m, kind, verts, n_verts, &iptr, &ilist);
    int64_t cap = 64, nnz = 0;
    int32_t* buf = xmalloc(sizeof(int32_t) * cap);
    if (rowptr) rowptr[0] = 0;
    for (int32_t i = 0; i < m; ++i) {
        int64_t cnt = 0;
        for (int k = 0; k < kind; ++k) {
            int32_t v = verts[(int64_t)i * kind + k];
            for (int64_t e = iptr[v]; e < iptr[v + 1]; ++e) {
                if (ilist[e] == i) continue;
                if (cnt == cap) { cap *= 2; buf = realloc(buf, sizeof(int32_t) * cap); if (!buf) abort(); }
                buf[cnt++] = ilist[e];
            }
        }
        qsort(buf, (size_t)cnt, sizeof(int32_t), cmp_i32);
        int64_t u = 0;
        for (int64_t e = 0; e < cnt; ++e)
            if (u == 0 || buf[e] != buf[u - 1]) buf[u++] = buf[e];
        if (col) {
            for (int64_t e = 0; e < u; ++e) col[nnz + e] = buf[e];
            col[nnz + u] = i; /* diagonal last */
        }
        nnz += u + 1;
        if (rowptr) rowptr[i + 1] = nnz;
    }
    free(buf); free(iptr); free(ilist);
    return nnz;
}

/* A = grad C M^-1 grad C^T + alpha_tilde (Eq. 3):
 * A_ii = sum_k w_{v_k} |g_{i,k}|^2 + alpha_tilde_i;
 * A_ij = sum over ALL shared vertices v (ascending id) of w_v g_{i,v} . g_{j,v} (reading c14). */
static void assemble_row(int32_t i, int kind, const int32_t* verts, const double* w, const double* g,
                         const double* alpha_tilde, const int64_t* rowptr, const int32_t* col, double* val) {
    const int32_t* vi = verts + (int64_t)i * kind;
    const double* gi = g + (int64_t)i * kind * 3;
    for (int64_t e = rowptr[i]; e < rowptr[i + 1] - 1; ++e) {
        int32_t j = col[e];
        const int32_t* vj = verts + (int64_t)j * kind;
        const double* gj = g + (int64_t)j * kind * 3;
        /* shared vertices in ascending vertex id */
        int32_t sv[4]; int ki[4], kj[4], ns = 0;
        for (int a = 0; a < kind; ++a)
            for (int b = 0; b < kind; ++b)
                if (vi[a] == vj[b]) { sv[ns] = vi[a]; ki[ns] = a; kj[ns] = b; ++ns; }
        for (int a = 0; a < ns; ++a)
            for (int b = a + 1; b < ns; ++b)
                if (sv[b] < sv[a]) {
                    int32_t t = sv[a]; sv[a] = sv[b]; sv[b] = t;
                    int u = ki[a]; ki[a] = ki[b]; ki[b] = u;
                    u = kj[a]; kj[a] = kj[b]; kj[b] = u;
                }
        double s = 0.0;
        for (int a = 0; a < ns; ++a) {
            const double* x1 = gi + 3 * ki[a];
            const double* x2 = gj + 3 * kj[a];
            s += w[sv[a]] * (x1[0] * x2[0] + x1[1] * x2[1] + x1[2] * x2[2]);
        }
        val[e] = s;
    }
    double d = 0.0;
    for (int k = 0; k < kind; ++k) {
        const double* x1 = gi + 3 * k;
        d += w[vi[k]] * (x1[0] * x1[0] + x1[1] * x1[1] + x1[2] * x1[2]);
    }
    val[rowptr[i + 1] - 1] = d + alpha_tilde[i];
}

void orc_assemble(int32_t m, int kind, const int32_t* verts, const double* w, const double* g,
                  const double* alpha_tilde, const int64_t* rowptr, const int32_t* col, double* val) {
    for (int32_t i = 0; i < m; ++i) assemble_row(i, kind, verts, w, g, alpha_tilde, rowptr, col, val);
}

/* The same definition restricted to the listed rows (sampled full-size parity checks). */
void orc_assemble_rows(int32_t nrows, const int32_t* rows, int kind, const int32_t* verts, const double* w,
                       const double* g, const double* alpha_tilde, const int64_t* rowptr, const int32_t* col,
                       double* val) {
    for (int32_t t = 0; t < nrows; ++t) assemble_row(rows[t], kind, verts, w, g, alpha_tilde, rowptr, col, val);
}

/* b = -C - alpha_tilde lambda (Eq. 3; Alg. 1 l.6). */
void orc_rhs(int32_t m, const double* C, const double* alpha_tilde, const double* lambda, double* b) {
    for (int32_t j = 0; j < m; ++j) b[j] = -C[j] - alpha_tilde[j] * lambda[j];
}

/* dx = M^-1 grad C^T dlambda (Eq. 5); per-vertex sum in ascending constraint order. */
void orc_apply_dx(int32_t m, int kind, const int32_t* verts, int32_t n_verts, const double* w,
                  const double* g, const double* dlambda, double* dx) {
    memset(dx, 0, sizeof(double) * 3 * (size_t)n_verts);
    for (int32_t j = 0; j < m; ++j)
        for (int k = 0; k < kind; ++k) {
            int32_t v = verts[(int64_t)j * kind + k];
            const double* gj = g + ((int64_t)j * kind + k) * 3;
            for (int r = 0; r < 3; ++r) dx[3 * (int64_t)v + r] += w[v] * gj[r] * dlambda[j];
        }
}

void orc_spmv(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val,
              const double* x, double* y) {
    for (int32_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) s += val[e] * x[col[e]];
        y[i] = s;
    }
}

/* ------------------------------------------------------------------------------------------
 * Setup (a3-a8), Fig. setup-pipline caption PAPER.md:241 and §4.1 PAPER.md:250-251.
 * ------------------------------------------------------------------------------------------ */

/* Filter: keep (i,j), i != j, iff |A_ij| >= theta sqrt(|A_ii||A_jj|) (c4). */
void orc_soc(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val, double theta,
             uint8_t* strong) {
    for (int32_t i = 0; i < n; ++i) {
        double aii = fabs(val[rowptr[i + 1] - 1]);
        for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
            int32_t j = col[e];
            if (j == i) { strong[e] = 0; continue; }
            double ajj = fabs(val[rowptr[j + 1] - 1]);
            strong[e] = fabs(val[e]) >= theta * sqrt(aii * ajj) ? 1 : 0;
        }
    }
}

typedef struct { uint64_t key; int32_t i; } keyed;
static int cmp_keyed(const void* a, const void* b) {
    const keyed* x = a; const keyed* y = b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return (x->i > y->i) - (x->i < y->i);
}
static keyed* priority_order(int32_t n, uint64_t seed, int stream, int level) {
    keyed* o = xmalloc(sizeof(keyed) * (size_t)n);
    for (int32_t i = 0; i < n; ++i) { o[i].key = orc_key(seed, stream, level, (uint64_t)i); o[i].i = i; }
    qsort(o, (size_t)n, sizeof(keyed), cmp_keyed);
    return o;
}

/* Aggregate (readings c2, c3).  Pass 1: visit nodes in ascending (key, i); a node
 * whose S-neighbourhood (itself included) is entirely unaggregated becomes a seed and claims
 * itself and its S-neighbours.  Ids = rank of the seed by node index.  Pass 2 (on a snapshot of
 * pass 1): each leftover joins the aggregate of its strong neighbour j with the largest |A_ij|
 * among pass-1-assigned neighbours, ties to the lowest aggregate id.  Returns n_agg. */
int32_t orc_aggregate(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val,
                      const uint8_t* strong, uint64_t seed, int level, int32_t* agg) {
    keyed* ord = priority_order(n, seed, 1, level);
    int32_t* lab = xmalloc(sizeof(int32_t) * (size_t)n);
    for (int32_t i = 0; i < n; ++i) lab[i] = -1;
    for (int32_t t = 0; t < n; ++t) {
        int32_t i = ord[t].i;
        if (lab[i] != -1) continue;
        int free_all = 1;
        for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e)
            if (strong[e] && lab[col[e]] != -1) { free_all = 0; break; }
        if (!free_all) continue;
        lab[i] = i;
        for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e)
            if (strong[e]) lab[col[e]] = i;
    }
    free(ord);
    /* ids by seed node index */
    int32_t* id = xmalloc(sizeof(int32_t) * (size_t)n);
    int32_t n_agg = 0;
    for (int32_t i = 0; i < n; ++i) id[i] = (lab[i] == i) ? n_agg++ : -1;
    int32_t* p1 = xmalloc(sizeof(int32_t) * (size_t)n);
    for (int32_t i = 0; i < n; ++i) p1[i] = lab[i] >= 0 ? id[lab[i]] : -1;
    for (int32_t i = 0; i < n; ++i) {
        if (p1[i] >= 0) { agg[i] = p1[i]; continue; }
        double best = -1.0; int32_t ba = -1;
        for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
            if (!strong[e]) continue;
            int32_t a = p1[col[e]];
            if (a < 0) continue;
            double s = fabs(val[e]);
            if (s > best || (s == best && a < ba)) { best = s; ba = a; }
        }
        agg[i] = ba; /* every leftover has one: pass 1 is maximal on S^2 */
    }
    free(lab); free(id); free(p1);
    return n_agg;
}

/* Colouring for the GS bootstrap (reading c5): greedy first-fit distance-1 colouring of the
 * pattern of A_0, visiting nodes in ascending (key(stream 2), i).  Returns #colours. */
int32_t orc_colour(int32_t n, const int64_t* rowptr, const int32_t* col, uint64_t seed, int32_t* colour) {
    keyed* ord = priority_order(n, seed, 2, 0);
    for (int32_t i = 0; i < n; ++i) colour[i] = -1;
    int32_t ncol = 0, cap = 64;
    uint8_t* used = xcalloc((size_t)cap, 1);
    for (int32_t t = 0; t < n; ++t) {
        int32_t i = ord[t].i;
        memset(used, 0, (size_t)cap);
        for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
            int32_t c = colour[col[e]];
            if (col[e] == i || c < 0) continue;
            while (c >= cap) { used = realloc(used, (size_t)cap * 2); memset(used + cap, 0, (size_t)cap); cap *= 2; }
            used[c] = 1;
        }
        int32_t c = 0;
        while (c < cap && used[c]) ++c;
        colour[i] = c;
        if (c + 1 > ncol) ncol = c + 1;
        if (ncol >= cap) { used = realloc(used, (size_t)cap * 2); memset(used + cap, 0, (size_t)cap); cap *= 2; }
    }
    free(used); free(ord);
    return ncol;
}

typedef struct { int32_t c, i; } ci_pair;
static int cmp_ci(const void* a, const void* b) {
    const ci_pair* x = a; const ci_pair* y = b;
    if (x->c != y->c) return (x->c > y->c) - (x->c < y->c);
    return (x->i > y->i) - (x->i < y->i);
}

/* Near-kernel bootstrap: `sweeps` Gauss-Seidel sweeps on A x = 0 from
 * x_0[i] = U(stream 3, 0, i) * max over all stored |A_ij| (reading c5).  GS visits nodes sorted by
 * (colour, index).  If ||B||_2 < 1e-14 sqrt(n), B = ones. */
void orc_gs_bootstrap(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val,
                      const int32_t* colour, int32_t sweeps, uint64_t seed, double* B) {
    double mx = 0.0;
    for (int64_t e = 0; e < rowptr[n]; ++e) mx = OMAX(mx, fabs(val[e]));
    for (int32_t i = 0; i < n; ++i) B[i] = orc_uniform(seed, 3, 0, (uint64_t)i) * mx;
    ci_pair* ord = xmalloc(sizeof(ci_pair) * (size_t)n);
    for (int32_t i = 0; i < n; ++i) { ord[i].c = colour[i]; ord[i].i = i; }
    qsort(ord, (size_t)n, sizeof(ci_pair), cmp_ci);
    for (int32_t s = 0; s < sweeps; ++s)
        for (int32_t t = 0; t < n; ++t) {
            int32_t i = ord[t].i;
            double acc = 0.0, d = 0.0;
            for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
                if (col[e] == i) d = val[e];
                else acc += val[e] * B[col[e]];
            }
            B[i] = -acc / d;
        }
    free(ord);
    double nn = 0.0;
    for (int32_t i = 0; i < n; ++i) nn += B[i] * B[i];
    if (sqrt(nn) < 1e-14 * sqrt((double)n))
        for (int32_t i = 0; i < n; ++i) B[i] = 1.0;
}

/* Inject (readings c1, c6) with k = 1: the thin QR of each aggregate's block
 * B_a is Q = B_a/||B_a||, R = ||B_a||.  P_i = B_i/||B_agg(i)||, B_next[a] = ||B_a||;
 * ||B_a|| = 0 => P_i = 1/sqrt(|a|), R = 0. */
void orc_prolongator(int32_t n, const int32_t* agg, int32_t n_agg, const double* B, double* P, double* B_next) {
    double* ss = xcalloc((size_t)n_agg, sizeof(double));
    int32_t* cnt = xcalloc((size_t)n_agg, sizeof(int32_t));
    for (int32_t i = 0; i < n; ++i) { ss[agg[i]] += B[i] * B[i]; cnt[agg[i]]++; }
    for (int32_t a = 0; a < n_agg; ++a) B_next[a] = sqrt(ss[a]);
    for (int32_t i = 0; i < n; ++i) {
        double nrm = B_next[agg[i]];
        P[i] = nrm > 0.0 ? B[i] / nrm : 1.0 / sqrt((double)cnt[agg[i]]);
    }
    free(ss); free(cnt);
}

/* Galerkin product A_{l+1} = P^T A_l P (Eq. 6): (A_{l+1})_{ab} =
 * sum_{i in a} sum_{j in b} P_i A_ij P_j, over stored entries of A_l; the coarse pattern is the
 * set of (agg i, agg j) over stored (i,j), off-diagonals ascending, diagonal last. */
int64_t orc_galerkin(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val,
                     const int32_t* agg, const double* P, int32_t n_agg,
                     int64_t* crowptr, int32_t* ccol, double* cval) {
    /* members of each aggregate, ascending */
    int64_t* mp = xcalloc((size_t)n_agg + 1, sizeof(int64_t));
    for (int32_t i = 0; i < n; ++i) mp[agg[i] + 1]++;
    for (int32_t a = 0; a < n_agg; ++a) mp[a + 1] += mp[a];
    int32_t* mem = xmalloc(sizeof(int32_t) * (size_t)n);
    int64_t* f = xmalloc(sizeof(int64_t) * ((size_t)n_agg + 1));
    memcpy(f, mp, sizeof(int64_t) * ((size_t)n_agg + 1));
    for (int32_t i = 0; i < n; ++i) mem[f[agg[i]]++] = i;
    free(f);
    double* acc = xcalloc((size_t)n_agg, sizeof(double));
    uint8_t* mark = xcalloc((size_t)n_agg, 1);
    int32_t* touched = xmalloc(sizeof(int32_t) * (size_t)n_agg);
    int64_t nnz = 0;
    if (crowptr) crowptr[0] = 0;
    for (int32_t a = 0; a < n_agg; ++a) {
        int32_t nt = 0;
        for (int64_t t = mp[a]; t < mp[a + 1]; ++t) {
            int32_t i = mem[t];
            for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
                int32_t b = agg[col[e]];
                if (!mark[b]) { mark[b] = 1; touched[nt++] = b; acc[b] = 0.0; }
                if (cval) acc[b] += P[i] * val[e] * P[col[e]];
            }
        }
        qsort(touched, (size_t)nt, sizeof(int32_t), cmp_i32);
        int32_t k = 0;
        for (int32_t t = 0; t < nt; ++t) {
            int32_t b = touched[t];
            if (b == a) continue;
            if (ccol) ccol[nnz + k] = b;
            if (cval) cval[nnz + k] = acc[b];
            ++k;
        }
        if (ccol) ccol[nnz + k] = a;
        if (cval) cval[nnz + k] = acc[a];
        nnz += k + 1;
        for (int32_t t = 0; t < nt; ++t) mark[touched[t]] = 0;
        if (crowptr) crowptr[a + 1] = nnz;
    }
    free(mp); free(mem); free(acc); free(mark); free(touched);
    return nnz;
}

/* ------------------------------------------------------------------------------------------
 * k > 1 near-kernel vectors ("We repeat this six times to generate
 * six distinct B"; "use QR decomposition to form the next level, where R of QR
 * decomposition serves as B at the next level").  Readings c23-c25.
 * ------------------------------------------------------------------------------------------ */

/* k bootstrapped columns (reading c23): column c is orc_gs_bootstrap's sweep sequence
 * from x_0[i] = U(stream 3, 0, i + c n) * max|A_ij| (reading c0: index offset c n per column), each
 * column with its own ||.|| < 1e-14 sqrt(n) => ones fallback.  B is column-major, B[c n + i]. */
void orc_gs_bootstrap_k(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val,
                        const int32_t* colour, int32_t sweeps, uint64_t seed, int32_t k, double* B) {
    double mx = 0.0;
    for (int64_t e = 0; e < rowptr[n]; ++e) mx = OMAX(mx, fabs(val[e]));
    ci_pair* ord = xmalloc(sizeof(ci_pair) * (size_t)n);
    for (int32_t i = 0; i < n; ++i) { ord[i].c = colour[i]; ord[i].i = i; }
    qsort(ord, (size_t)n, sizeof(ci_pair), cmp_ci);
    for (int32_t c = 0; c < k; ++c) {
        double* x = B + (int64_t)c * n;
        for (int32_t i = 0; i < n; ++i) x[i] = orc_uniform(seed, 3, 0, (uint64_t)i + (uint64_t)c * (uint64_t)n) * mx;
        for (int32_t s = 0; s < sweeps; ++s)
            for (int32_t t = 0; t < n; ++t) {
                int32_t i = ord[t].i;
                double acc = 0.0, d = 0.0;
                for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
                    if (col[e] == i) d = val[e];
                    else acc += val[e] * x[col[e]];
                }
                x[i] = -acc / d;
            }
        double nn = 0.0;
        for (int32_t i = 0; i < n; ++i) nn += x[i] * x[i];
        if (sqrt(nn) < 1e-14 * sqrt((double)n))
            for (int32_t i = 0; i < n; ++i) x[i] = 1.0;
    }
    free(ord);
}

/* Inject with k columns (readings c24, c25).  For each aggregate a (members N_a
 * ascending) the |N_a| x k block B_a = B[N_a, :] is factored B_a = Q_a R_a by modified Gram-Schmidt
 * with one re-orthogonalisation pass, columns in order 0..k-1: column c is kept iff the norm of its
 * component orthogonal to the kept columns exceeds rank_tol * ||B_a[:, c]|| (and is > 0); kept columns
 * get R diagonal = that norm > 0, dropped (rank-deficient) columns only their projections.  Q_a fills
 * P's rows N_a in r_a consecutive coarse columns off_a .. off_a + r_a - 1 (off = prefix sum of r);
 * row j of R_a (r_a x k) becomes row off_a + j of B_next (n_next x k, column-major with leading
 * dimension ld_next).  An aggregate with no kept column (B_a = 0) gets the single column
 * 1/sqrt(|N_a|) with a zero R row (the k = 1 rule of reading c6).  P is CSR (pptr n+1, pcol, pval;
 * row i holds r_agg(i) entries, ascending columns).  B is column-major n x k.  Returns n_next; coff
 * (n_agg + 1) receives the offsets.  With pcol == NULL only coff / n_next are computed. */
int32_t orc_prolongator_qr(int32_t n, const int32_t* agg, int32_t n_agg, int32_t k, const double* B,
                           double rank_tol, int32_t* coff, int64_t* pptr, int32_t* pcol, double* pval,
                           double* B_next, int32_t ld_next) {
    int64_t* mp = xcalloc((size_t)n_agg + 1, sizeof(int64_t));
    for (int32_t i = 0; i < n; ++i) mp[agg[i] + 1]++;
    for (int32_t a = 0; a < n_agg; ++a) mp[a + 1] += mp[a];
    int32_t* mem = xmalloc(sizeof(int32_t) * (size_t)n);
    int64_t* f = xmalloc(sizeof(int64_t) * ((size_t)n_agg + 1));
    memcpy(f, mp, sizeof(int64_t) * ((size_t)n_agg + 1));
    for (int32_t i = 0; i < n; ++i) mem[f[agg[i]]++] = i;
    free(f);
    int32_t maxm = 0;
    for (int32_t a = 0; a < n_agg; ++a) maxm = (int32_t)OMAX(maxm, mp[a + 1] - mp[a]);
    double* Q = xmalloc(sizeof(double) * (size_t)maxm * (size_t)k);   /* kept columns, |N_a| each */
    double* v = xmalloc(sizeof(double) * (size_t)maxm);
    double* R = xmalloc(sizeof(double) * (size_t)k * (size_t)k);     /* R[j*k + c] */
    double* Qs = pval ? xmalloc(sizeof(double) * (size_t)n * (size_t)k) : NULL;  /* Q by member slot */
    int32_t* rk = xmalloc(sizeof(int32_t) * (size_t)n_agg);
    coff[0] = 0;
    for (int32_t a = 0; a < n_agg; ++a) {
        const int64_t m0 = mp[a];
        const int32_t na = (int32_t)(mp[a + 1] - m0);
        int32_t r = 0;
        memset(R, 0, sizeof(double) * (size_t)k * (size_t)k);
        for (int32_t c = 0; c < k; ++c) {
            double bn = 0.0;
            for (int32_t t = 0; t < na; ++t) { v[t] = B[(int64_t)c * n + mem[m0 + t]]; bn += v[t] * v[t]; }
            bn = sqrt(bn);
            for (int pass = 0; pass < 2; ++pass)
                for (int32_t j = 0; j < r; ++j) {
                    double s = 0.0;
                    for (int32_t t = 0; t < na; ++t) s += Q[(int64_t)j * na + t] * v[t];
                    for (int32_t t = 0; t < na; ++t) v[t] -= s * Q[(int64_t)j * na + t];
                    R[j * k + c] += s;
                }
            double vn = 0.0;
            for (int32_t t = 0; t < na; ++t) vn += v[t] * v[t];
            vn = sqrt(vn);
            if (vn > 0.0 && vn > rank_tol * bn) {
                for (int32_t t = 0; t < na; ++t) Q[(int64_t)r * na + t] = v[t] / vn;
                R[r * k + c] = vn;
                ++r;
            }
        }
        if (r == 0) {   /* B_a = 0: uniform column, zero R row (reading c6) */
            for (int32_t t = 0; t < na; ++t) Q[t] = 1.0 / sqrt((double)na);
            memset(R, 0, sizeof(double) * (size_t)k);
            r = 1;
        }
        rk[a] = r;
        coff[a + 1] = coff[a] + r;
        if (B_next)
            for (int32_t j = 0; j < r; ++j)
                for (int32_t c = 0; c < k; ++c) B_next[(int64_t)c * ld_next + coff[a] + j] = R[j * k + c];
        if (Qs)
            for (int32_t j = 0; j < r; ++j)
                for (int32_t t = 0; t < na; ++t) Qs[(int64_t)(m0 + t) * k + j] = Q[(int64_t)j * na + t];
    }
    if (pptr) {
        pptr[0] = 0;
        for (int32_t i = 0; i < n; ++i) pptr[i + 1] = pptr[i] + rk[agg[i]];
    }
    if (pcol && pval) {
        for (int32_t a = 0; a < n_agg; ++a)
            for (int64_t t = mp[a]; t < mp[a + 1]; ++t) {
                const int32_t i = mem[t];
                for (int32_t j = 0; j < rk[a]; ++j) {
                    pcol[pptr[i] + j] = coff[a] + j;
                    pval[pptr[i] + j] = Qs[t * k + j];
                }
            }
    }
    const int32_t nn = coff[n_agg];
    free(mp); free(mem); free(Q); free(v); free(R); free(Qs); free(rk);
    return nn;
}

/* Galerkin product A_c = P^T A P for a general CSR prolongator (Eq. 6; used with
 * k > 1): (A_c)_{IJ} = sum_i sum_{j in row i of A} P_{iI} A_ij P_{jJ}.  Coarse row I accumulates over
 * the fine rows i with P_{iI} != 0 in ascending i, their stored entries in storage order, and P's
 * row j in storage order; the pattern is every (I, J) reached, off-diagonals ascending, diagonal
 * last.  All-NULL outputs => count only (returns nnz). */
int64_t orc_galerkin_p(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val,
                       const int64_t* pptr, const int32_t* pcol, const double* pval, int32_t nc,
                       int64_t* crowptr, int32_t* ccol, double* cval) {
    /* P^T by coarse column: fine rows ascending */
    int64_t* tp = xcalloc((size_t)nc + 1, sizeof(int64_t));
    for (int64_t e = 0; e < pptr[n]; ++e) tp[pcol[e] + 1]++;
    for (int32_t I = 0; I < nc; ++I) tp[I + 1] += tp[I];
    int32_t* ti = xmalloc(sizeof(int32_t) * (size_t)OMAX(pptr[n], 1));
    double* tv = xmalloc(sizeof(double) * (size_t)OMAX(pptr[n], 1));
    int64_t* f = xmalloc(sizeof(int64_t) * ((size_t)nc + 1));
    memcpy(f, tp, sizeof(int64_t) * ((size_t)nc + 1));
    for (int32_t i = 0; i < n; ++i)
        for (int64_t e = pptr[i]; e < pptr[i + 1]; ++e) { ti[f[pcol[e]]] = i; tv[f[pcol[e]]++] = pval[e]; }
    free(f);
    double* acc = xcalloc((size_t)nc, sizeof(double));
    uint8_t* mark = xcalloc((size_t)nc, 1);
    int32_t* touched = xmalloc(sizeof(int32_t) * (size_t)nc);
    int64_t nnz = 0;
    if (crowptr) crowptr[0] = 0;
    for (int32_t I = 0; I < nc; ++I) {
        int32_t nt = 0;
        for (int64_t t = tp[I]; t < tp[I + 1]; ++t) {
            const int32_t i = ti[t];
            const double pi = tv[t];
            for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
                const int32_t j = col[e];
                for (int64_t q = pptr[j]; q < pptr[j + 1]; ++q) {
                    const int32_t J = pcol[q];
                    if (!mark[J]) { mark[J] = 1; touched[nt++] = J; acc[J] = 0.0; }
                    if (cval) acc[J] += pi * val[e] * pval[q];
                }
            }
        }
        qsort(touched, (size_t)nt, sizeof(int32_t), cmp_i32);
        int32_t k = 0;
        for (int32_t t = 0; t < nt; ++t) {
            const int32_t J = touched[t];
            if (J == I) continue;
            if (ccol) ccol[nnz + k] = J;
            if (cval) cval[nnz + k] = acc[J];
            ++k;
        }
        if (ccol) ccol[nnz + k] = I;
        if (cval) cval[nnz + k] = mark[I] ? acc[I] : 0.0;
        nnz += k + 1;
        for (int32_t t = 0; t < nt; ++t) mark[touched[t]] = 0;
        if (crowptr) crowptr[I + 1] = nnz;
    }
    free(tp); free(ti); free(tv); free(acc); free(mark); free(touched);
    return nnz;
}

/* lambda_max(D^-1 A) by the power method (reading c9): v_0 = U(stream 4, l)/||.||;
 * `iters` times: w = D^-1 A v; lambda = ||w||_2; v = w / lambda. */
/* `iters` power iterations from the normalised vector v (updated in place: the last normalised iterate). */
double orc_power_from(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val, int32_t iters,
                      double* v) {
    double* w = xmalloc(sizeof(double) * (size_t)n);
    double lam = 0.0;
    for (int32_t it = 0; it < iters; ++it) {
        orc_spmv(n, rowptr, col, val, v, w);
        double s = 0.0;
        for (int32_t i = 0; i < n; ++i) { w[i] /= val[rowptr[i + 1] - 1]; s += w[i] * w[i]; }
        lam = sqrt(s);
        if (lam == 0.0) break;
        for (int32_t i = 0; i < n; ++i) v[i] = w[i] / lam;
    }
    free(w);
    return lam;
}

static void power_start(int32_t n, uint64_t seed, int level, double* v) {
    double nn = 0.0;
    for (int32_t i = 0; i < n; ++i) { v[i] = orc_uniform(seed, 4, level, (uint64_t)i); nn += v[i] * v[i]; }
    nn = sqrt(nn);
    for (int32_t i = 0; i < n; ++i) v[i] /= nn;
}

double orc_power(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val,
                 int32_t iters, uint64_t seed, int level) {
    double* v = xmalloc(sizeof(double) * (size_t)n);
    power_start(n, seed, level, v);
    const double lam = orc_power_from(n, rowptr, col, val, iters, v);
    free(v);
    return lam;
}

/* Dense Cholesky A = L L^T (coarsest solve; reading c8).  Returns -1 if not SPD. */
int orc_cholesky(int32_t n, const double* A, double* L) {
    memset(L, 0, sizeof(double) * (size_t)n * n);
    for (int32_t j = 0; j < n; ++j) {
        double s = A[(int64_t)j * n + j];
        for (int32_t k = 0; k < j; ++k) s -= L[(int64_t)j * n + k] * L[(int64_t)j * n + k];
        if (!(s > 0.0)) return -1;
        double d = sqrt(s);
        L[(int64_t)j * n + j] = d;
        for (int32_t i = j + 1; i < n; ++i) {
            double t = A[(int64_t)i * n + j];
            for (int32_t k = 0; k < j; ++k) t -= L[(int64_t)i * n + k] * L[(int64_t)j * n + k];
            L[(int64_t)i * n + j] = t / d;
        }
    }
    return 0;
}

void orc_chol_solve(int32_t n, const double* L, const double* b, double* x) {
    for (int32_t i = 0; i < n; ++i) {
        double s = b[i];
        for (int32_t k = 0; k < i; ++k) s -= L[(int64_t)i * n + k] * x[k];
        x[i] = s / L[(int64_t)i * n + i];
    }
    for (int32_t i = n - 1; i >= 0; --i) {
        double s = x[i];
        for (int32_t k = i + 1; k < n; ++k) s -= L[(int64_t)k * n + i] * x[k];
        x[i] = s / L[(int64_t)i * n + i];
    }
}

/* ------------------------------------------------------------------------------------------
 * Hierarchy + solve (a6-a11).
 * ------------------------------------------------------------------------------------------ */
typedef struct {
    int32_t n; int64_t nnz;
    int64_t* rowptr; int32_t* col; double* val;
    int32_t* agg; int32_t n_agg; double* P; double omega;
    double cheb_theta, cheb_delta;  /* Chebyshev interval (reading c20) */
    int32_t* gs_order;              /* multicolour GS: nodes sorted by (colour, index) (reading c22) */
    /* k > 1 (f2): general CSR prolongator n x n_next (row i: r_agg(i) entries), coarse offsets */
    int64_t* pptr; int32_t* pcol; double* pval; int32_t* coff;
    double* pw_v;                   /* last normalised power iterate of D^-1 A (omega refresh start) */
} orc_level;

struct orc_hier {
    int L;
    orc_level lv[32];
    double* Lc;          /* Cholesky factor of the coarsest matrix */
    double* B0;          /* bootstrapped near-kernel vector(s) at level 0 (if coarsened): n x k column-major */
    int32_t ncolours;
    int stalled;
    orc_config cfg;
};

static void level_free(orc_level* v) {
    free(v->rowptr); free(v->col); free(v->val); free(v->agg); free(v->P); free(v->gs_order);
    free(v->pptr); free(v->pcol); free(v->pval); free(v->coff); free(v->pw_v);
    memset(v, 0, sizeof *v);
}

static int factor_coarsest(orc_hier* h) {
    orc_level* c = &h->lv[h->L - 1];
    int32_t n = c->n;
    double* A = xcalloc((size_t)n * n, sizeof(double));
    for (int32_t i = 0; i < n; ++i)
        for (int64_t e = c->rowptr[i]; e < c->rowptr[i + 1]; ++e) A[(int64_t)i * n + c->col[e]] = c->val[e];
    free(h->Lc);
    h->Lc = xmalloc(sizeof(double) * (size_t)n * n);
    int rc = orc_cholesky(n, A, h->Lc);
    free(A);
    return rc;
}

/* Setup pipeline (§4.1): per level Filter -> Aggregate -> Inject -> Galerkin;
 * the level-0 near kernel comes from the GS bootstrap (§4.3), coarser ones from R (c6); omega_l
 * = 2/(s lambda_max(D^-1 A_l) + lambda_min_est) (§4.5; safety s, reading c9); stop when n < min_coarse (c7). */
orc_hier* orc_hier_build(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val,
                         const orc_config* cfg) {
    orc_hier* h = xcalloc(1, sizeof(orc_hier));
    h->cfg = *cfg;
    orc_level* l0 = &h->lv[0];
    l0->n = n; l0->nnz = rowptr[n];
    l0->rowptr = xmalloc(sizeof(int64_t) * ((size_t)n + 1));
    l0->col = xmalloc(sizeof(int32_t) * (size_t)l0->nnz);
    l0->val = xmalloc(sizeof(double) * (size_t)l0->nnz);
    memcpy(l0->rowptr, rowptr, sizeof(int64_t) * ((size_t)n + 1));
    memcpy(l0->col, col, sizeof(int32_t) * (size_t)l0->nnz);
    memcpy(l0->val, val, sizeof(double) * (size_t)l0->nnz);
    h->L = 1;
    double* B = NULL;
    const int32_t k = cfg->k_nullspace > 1 ? cfg->k_nullspace : 1;
    int maxl = cfg->max_levels < 32 ? cfg->max_levels : 32;
    for (int l = 0; l + 1 < maxl; ++l) {
        orc_level* a = &h->lv[l];
        if (a->n < cfg->min_coarse) break;
        uint8_t* S = xmalloc((size_t)a->nnz);
        orc_soc(a->n, a->rowptr, a->col, a->val, cfg->theta, S);
        int32_t* agg = xmalloc(sizeof(int32_t) * (size_t)a->n);
        int32_t na = orc_aggregate(a->n, a->rowptr, a->col, a->val, S, cfg->seed, l, agg);
        free(S);
        if ((double)na > cfg->stall_ratio * (double)a->n) { free(agg); h->stalled = 1; break; }
        if (l == 0) {
            int32_t* colour = xmalloc(sizeof(int32_t) * (size_t)a->n);
            h->ncolours = orc_colour(a->n, a->rowptr, a->col, cfg->seed, colour);
            B = xmalloc(sizeof(double) * (size_t)a->n * (size_t)k);
            if (k == 1) orc_gs_bootstrap(a->n, a->rowptr, a->col, a->val, colour, cfg->bootstrap_sweeps, cfg->seed, B);
            else orc_gs_bootstrap_k(a->n, a->rowptr, a->col, a->val, colour, cfg->bootstrap_sweeps, cfg->seed, k, B);
            free(colour);
            h->B0 = xmalloc(sizeof(double) * (size_t)a->n * (size_t)k);
            memcpy(h->B0, B, sizeof(double) * (size_t)a->n * (size_t)k);
        }
        a->agg = agg; a->n_agg = na;
        orc_level* c = &h->lv[l + 1];
        if (k == 1) {
            a->P = xmalloc(sizeof(double) * (size_t)a->n);
            double* Bn = xmalloc(sizeof(double) * (size_t)na);
            orc_prolongator(a->n, agg, na, B, a->P, Bn);
            free(B); B = Bn;
            c->n = na;
            c->rowptr = xmalloc(sizeof(int64_t) * ((size_t)na + 1));
            c->nnz = orc_galerkin(a->n, a->rowptr, a->col, a->val, agg, a->P, na, c->rowptr, NULL, NULL);
            c->col = xmalloc(sizeof(int32_t) * (size_t)c->nnz);
            c->val = xmalloc(sizeof(double) * (size_t)c->nnz);
            orc_galerkin(a->n, a->rowptr, a->col, a->val, agg, a->P, na, c->rowptr, c->col, c->val);
        } else {  /* k columns (f2): QR injection, general P^T A P on the scalar coarse DOFs (c24, c25) */
            a->coff = xmalloc(sizeof(int32_t) * ((size_t)na + 1));
            a->pptr = xmalloc(sizeof(int64_t) * ((size_t)a->n + 1));
            const int32_t nc = orc_prolongator_qr(a->n, agg, na, k, B, ORC_RANK_TOL, a->coff, a->pptr, NULL, NULL, NULL, 0);
            if ((double)nc > cfg->stall_ratio * (double)a->n) {  /* coarse DOFs, not aggregates, decide (c7) */
                free(a->coff); free(a->pptr); free(a->agg);
                a->coff = NULL; a->pptr = NULL; a->agg = NULL; a->n_agg = 0;
                h->stalled = 1;
                break;
            }
            a->pcol = xmalloc(sizeof(int32_t) * (size_t)a->pptr[a->n]);
            a->pval = xmalloc(sizeof(double) * (size_t)a->pptr[a->n]);
            double* Bn = xmalloc(sizeof(double) * (size_t)nc * (size_t)k);
            orc_prolongator_qr(a->n, agg, na, k, B, ORC_RANK_TOL, a->coff, a->pptr, a->pcol, a->pval, Bn, nc);
            free(B); B = Bn;
            c->n = nc;
            c->rowptr = xmalloc(sizeof(int64_t) * ((size_t)nc + 1));
            c->nnz = orc_galerkin_p(a->n, a->rowptr, a->col, a->val, a->pptr, a->pcol, a->pval, nc, c->rowptr, NULL, NULL);
            c->col = xmalloc(sizeof(int32_t) * (size_t)c->nnz);
            c->val = xmalloc(sizeof(double) * (size_t)c->nnz);
            orc_galerkin_p(a->n, a->rowptr, a->col, a->val, a->pptr, a->pcol, a->pval, nc, c->rowptr, c->col, c->val);
        }
        a->pw_v = xmalloc(sizeof(double) * (size_t)a->n);
        power_start(a->n, cfg->seed, l, a->pw_v);
        double lam = orc_power_from(a->n, a->rowptr, a->col, a->val, cfg->power_iters, a->pw_v);
        a->omega = 2.0 / (cfg->lambda_safety * lam + cfg->lambda_min_est);
        if (cfg->smoother == 2) {  /* multicolour GS order of this level (reading c22) */
            int32_t* colour = xmalloc(sizeof(int32_t) * (size_t)a->n);
            orc_colour(a->n, a->rowptr, a->col, cfg->seed, colour);
            ci_pair* ord = xmalloc(sizeof(ci_pair) * (size_t)a->n);
            for (int32_t i = 0; i < a->n; ++i) { ord[i].c = colour[i]; ord[i].i = i; }
            qsort(ord, (size_t)a->n, sizeof(ci_pair), cmp_ci);
            a->gs_order = xmalloc(sizeof(int32_t) * (size_t)a->n);
            for (int32_t i = 0; i < a->n; ++i) a->gs_order[i] = ord[i].i;
            free(ord); free(colour);
        }
        {   /* Chebyshev interval [cheb_lower*hi, hi], hi = safety*lambda_max (reading c20) */
            const double hi = cfg->lambda_safety * lam, lo = cfg->cheb_lower * hi;
            a->cheb_theta = 0.5 * (hi + lo);
            a->cheb_delta = 0.5 * (hi - lo);
        }
        h->L = l + 2;
    }
    free(B);
    factor_coarsest(h);
    return h;
}

/* Smoother parameters of every level from `iters` further power iterations on the CURRENT level matrices,
 * started from the last normalised iterate (reading c26: the optional per-frame omega refresh).  Same formulas
 * as orc_hier_build. */
static void set_smoother_params(orc_level* a, const orc_config* cfg, double lam) {
    a->omega = 2.0 / (cfg->lambda_safety * lam + cfg->lambda_min_est);
    const double hi = cfg->lambda_safety * lam, lo = cfg->cheb_lower * hi;
    a->cheb_theta = 0.5 * (hi + lo);
    a->cheb_delta = 0.5 * (hi - lo);
}
void orc_hier_refresh_omega(orc_hier* h, int32_t iters) {
    if (iters <= 0) return;
    for (int l = 0; l + 1 < h->L; ++l) {
        orc_level* a = &h->lv[l];
        if (!a->pw_v) continue;
        const double lam = orc_power_from(a->n, a->rowptr, a->col, a->val, iters, a->pw_v);
        set_smoother_params(a, &h->cfg, lam);
    }
}

/* Solving phase: recompute A_{l+1} = P_l^T A_l P_l with the cached P (values of the
 * current A_0), then refactor the coarsest matrix.  Returns -1 if the coarsest is not SPD. */
int orc_hier_refresh(orc_hier* h, const double* val0) {
    memcpy(h->lv[0].val, val0, sizeof(double) * (size_t)h->lv[0].nnz);
    for (int l = 0; l + 1 < h->L; ++l) {
        orc_level* a = &h->lv[l]; orc_level* c = &h->lv[l + 1];
        if (a->pptr) orc_galerkin_p(a->n, a->rowptr, a->col, a->val, a->pptr, a->pcol, a->pval, c->n, c->rowptr, c->col, c->val);
        else orc_galerkin(a->n, a->rowptr, a->col, a->val, a->agg, a->P, a->n_agg, c->rowptr, c->col, c->val);
    }
    return factor_coarsest(h);
}

void orc_hier_free(orc_hier* h) {
    if (!h) return;
    for (int l = 0; l < h->L; ++l) level_free(&h->lv[l]);
    free(h->Lc); free(h->B0); free(h);
}
int orc_hier_levels(const orc_hier* h) { return h->L; }
void orc_hier_level_size(const orc_hier* h, int l, int32_t* n, int64_t* nnz) { *n = h->lv[l].n; *nnz = h->lv[l].nnz; }
void orc_hier_get_level(const orc_hier* h, int l, int64_t* rowptr, int32_t* col, double* val) {
    const orc_level* a = &h->lv[l];
    if (rowptr) memcpy(rowptr, a->rowptr, sizeof(int64_t) * ((size_t)a->n + 1));
    if (col) memcpy(col, a->col, sizeof(int32_t) * (size_t)a->nnz);
    if (val) memcpy(val, a->val, sizeof(double) * (size_t)a->nnz);
}
void orc_hier_get_agg(const orc_hier* h, int l, int32_t* agg) { memcpy(agg, h->lv[l].agg, sizeof(int32_t) * (size_t)h->lv[l].n); }
void orc_hier_get_P(const orc_hier* h, int l, double* P) { if (h->lv[l].P) memcpy(P, h->lv[l].P, sizeof(double) * (size_t)h->lv[l].n); }
double orc_hier_omega(const orc_hier* h, int l) { return h->lv[l].omega; }
void orc_hier_get_B0(const orc_hier* h, double* B) {
    const size_t k = h->cfg.k_nullspace > 1 ? (size_t)h->cfg.k_nullspace : 1;
    if (h->B0) memcpy(B, h->B0, sizeof(double) * (size_t)h->lv[0].n * k);
}
/* level-l prolongator as CSR (n_l x n_{l+1}); k = 1 levels are returned in the same form (one entry per
 * row, column = aggregate).  rowptr == NULL: only *nnz. */
void orc_hier_get_P_csr(const orc_hier* h, int l, int64_t* nnz, int64_t* rowptr, int32_t* col, double* val) {
    const orc_level* a = &h->lv[l];
    if (a->pptr) {
        *nnz = a->pptr[a->n];
        if (rowptr) memcpy(rowptr, a->pptr, sizeof(int64_t) * ((size_t)a->n + 1));
        if (col) memcpy(col, a->pcol, sizeof(int32_t) * (size_t)*nnz);
        if (val) memcpy(val, a->pval, sizeof(double) * (size_t)*nnz);
        return;
    }
    *nnz = a->n;
    for (int32_t i = 0; i < a->n; ++i) {
        if (rowptr) rowptr[i] = i;
        if (col) col[i] = a->agg[i];
        if (val) val[i] = a->P[i];
    }
    if (rowptr) rowptr[a->n] = a->n;
}
int32_t orc_hier_n_colours(const orc_hier* h) { return h->ncolours; }

/* omega-Jacobi sweep x <- x + omega D^-1 (b - A x). */
static void jacobi(const orc_level* a, const double* b, double* x, double* tmp) {
    orc_spmv(a->n, a->rowptr, a->col, a->val, x, tmp);
    for (int32_t i = 0; i < a->n; ++i) x[i] += a->omega * (b[i] - tmp[i]) / a->val[a->rowptr[i + 1] - 1];
}

/* Chebyshev smoother (lazily set parameters PAPER.md:320; reading c20): `sweeps` steps
 * of the Chebyshev iteration for A x = b preconditioned by D = diag(A) on the interval
 * [lo, hi] of D^-1 A (Saad, Iterative Methods for Sparse Linear Systems, 2nd ed., Alg. 12.1):
 *   theta = (hi+lo)/2, delta = (hi-lo)/2, sigma = theta/delta, rho_0 = 1/sigma,
 *   step 0:  r = D^-1 (b - A x),  d = r / theta,                                   x += d
 *   step k:  r = D^-1 (b - A x),  rho_k = 1/(2 sigma - rho_{k-1}),
 *            d = rho_k rho_{k-1} d + (2 rho_k / delta) r,                            x += d        */
static void chebyshev(const orc_level* a, int sweeps, const double* b, double* x, double* tmp, double* d) {
    const double theta = a->cheb_theta, delta = a->cheb_delta, sigma = theta / delta;
    double rho = 1.0 / sigma;
    for (int k = 0; k < sweeps; ++k) {
        orc_spmv(a->n, a->rowptr, a->col, a->val, x, tmp);
        const double rho_new = k == 0 ? rho : 1.0 / (2.0 * sigma - rho);
        for (int32_t i = 0; i < a->n; ++i) {
            const double r = (b[i] - tmp[i]) / a->val[a->rowptr[i + 1] - 1];
            d[i] = k == 0 ? r / theta : rho_new * rho * d[i] + (2.0 * rho_new / delta) * r;
            x[i] += d[i];
        }
        rho = rho_new;
    }
}

/* Multicolour Gauss-Seidel ("parallel GS"; reading c22): one sweep updates the nodes in
 * (colour, index) order — forward for pre-smoothing, reversed for post-smoothing, so the V-cycle stays
 * symmetric: x_i = (b_i - sum_{j != i} A_ij x_j) / A_ii with the latest x. */
static void gauss_seidel(const orc_level* a, int sweeps, int backward, const double* b, double* x) {
    for (int s = 0; s < sweeps; ++s)
        for (int32_t t = 0; t < a->n; ++t) {
            const int32_t i = a->gs_order[backward ? a->n - 1 - t : t];
            double acc = 0.0, dg = 0.0;
            for (int64_t e = a->rowptr[i]; e < a->rowptr[i + 1]; ++e) {
                if (a->col[e] == i) dg = a->val[e];
                else acc += a->val[e] * x[a->col[e]];
            }
            x[i] = (b[i] - acc) / dg;
        }
}

static void smooth(const orc_hier* h, const orc_level* a, const double* b, double* x, double* tmp, double* d,
                   int post) {
    if (h->cfg.smoother == 1) chebyshev(a, h->cfg.smoother_sweeps, b, x, tmp, d);
    else if (h->cfg.smoother == 2) gauss_seidel(a, h->cfg.smoother_sweeps, post, b, x);
    else for (int s = 0; s < h->cfg.smoother_sweeps; ++s) jacobi(a, b, x, tmp);
}

void orc_hier_cheb(const orc_hier* h, int l, double* theta, double* delta) {
    *theta = h->lv[l].cheb_theta; *delta = h->lv[l].cheb_delta;
}
void orc_hier_smooth(const orc_hier* h, int l, const double* b, double* x, int post) {
    const orc_level* a = &h->lv[l];
    double* tmp = xmalloc(sizeof(double) * (size_t)a->n);
    double* d = xmalloc(sizeof(double) * (size_t)a->n);
    smooth(h, a, b, x, tmp, d, post);
    free(tmp); free(d);
}

/* V-cycle from x = 0: nu pre-sweeps, r = b - A x, b_c = P^T r, recurse,
 * x += P e, nu post-sweeps; coarsest level solved by the dense Cholesky factor (c8). */
static void vcycle_level(const orc_hier* h, int l, const double* b, double* x) {
    const orc_level* a = &h->lv[l];
    if (l == h->L - 1) { orc_chol_solve(a->n, h->Lc, b, x); return; }
    int32_t n = a->n, nc = h->lv[l + 1].n;
    double* tmp = xmalloc(sizeof(double) * (size_t)n);
    double* d = xmalloc(sizeof(double) * (size_t)n);
    for (int32_t i = 0; i < n; ++i) x[i] = 0.0;
    smooth(h, a, b, x, tmp, d, 0);
    orc_spmv(n, a->rowptr, a->col, a->val, x, tmp);
    double* bc = xcalloc((size_t)nc, sizeof(double));
    double* ec = xmalloc(sizeof(double) * (size_t)nc);
    if (a->pptr) {   /* general P (k > 1): b_c = P^T r, x += P e */
        for (int32_t i = 0; i < n; ++i)
            for (int64_t q = a->pptr[i]; q < a->pptr[i + 1]; ++q) bc[a->pcol[q]] += a->pval[q] * (b[i] - tmp[i]);
        vcycle_level(h, l + 1, bc, ec);
        for (int32_t i = 0; i < n; ++i)
            for (int64_t q = a->pptr[i]; q < a->pptr[i + 1]; ++q) x[i] += a->pval[q] * ec[a->pcol[q]];
    } else {
        for (int32_t i = 0; i < n; ++i) bc[a->agg[i]] += a->P[i] * (b[i] - tmp[i]);
        vcycle_level(h, l + 1, bc, ec);
        for (int32_t i = 0; i < n; ++i) x[i] += a->P[i] * ec[a->agg[i]];
    }
    smooth(h, a, b, x, tmp, d, 1);
    free(tmp); free(d); free(bc); free(ec);
}

void orc_vcycle(const orc_hier* h, const double* b, double* x) { vcycle_level(h, 0, b, x); }

static double dot(int32_t n, const double* a, const double* b) {
    double s = 0.0;
    for (int32_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

/* MGPCG (Alg. 1 l.8) with a fixed iteration count (reading c10), x_0 = 0.
 * Guards: alpha = 0 if p.q == 0; beta = 0 if the previous r.z == 0.  Returns the number of
 * iterations with <z,r> < 0 or (<z,r> == 0 and r != 0) (indefinite preconditioner). */
int orc_pcg(const orc_hier* h, const double* b, int32_t iters, double* x, double* rz_trace) {
    const orc_level* a = &h->lv[0];
    int32_t n = a->n;
    double* r = xmalloc(sizeof(double) * (size_t)n);
    double* z = xmalloc(sizeof(double) * (size_t)n);
    double* p = xcalloc((size_t)n, sizeof(double));
    double* q = xmalloc(sizeof(double) * (size_t)n);
    int rc = 0;
    for (int32_t i = 0; i < n; ++i) { x[i] = 0.0; r[i] = b[i]; }
    double rz_old = 0.0;
    const double tol = h->cfg.pcg_tol, bb = dot(n, b, b);
    for (int32_t k = 0; k < iters; ++k) {
        /* optional convergence exit (reading c10: off by default): stop before iteration k once the
         * residual r_k meets ||r_k|| <= pcg_tol ||b|| */
        if (tol > 0.0 && sqrt(dot(n, r, r)) <= tol * sqrt(bb)) break;
        orc_vcycle(h, r, z);
        double rz = dot(n, r, z);
        if (rz_trace) rz_trace[k] = rz;
        if (rz < 0.0 || (rz == 0.0 && dot(n, r, r) > 0.0)) rc++;
        double beta = (k == 0 || rz_old == 0.0) ? 0.0 : rz / rz_old;
        for (int32_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
        orc_spmv(n, a->rowptr, a->col, a->val, p, q);
        double pq = dot(n, p, q);
        double alpha = pq != 0.0 ? rz / pq : 0.0;
        for (int32_t i = 0; i < n; ++i) { x[i] += alpha * p[i]; r[i] -= alpha * q[i]; }
        rz_old = rz;
    }
    free(r); free(z); free(p); free(q);
    return rc;
}

/* ------------------------------------------------------------------------------------------
 * Simulation loop, Algorithm 1.
 * ------------------------------------------------------------------------------------------ */
struct orc_sim {
    int kind; int32_t n, m;
    int32_t* verts;
    double *x, *v, *x_old, *w, *alpha;
    double *rest_len, *Dm_inv, *vol;
    double *C, *g, *lambda, *dl, *b, *atilde, *dx;
    int64_t* rowptr; int32_t* col; double* val; int64_t nnz;
    orc_hier* h;
    int64_t frame;
    int stale;
    orc_config cfg;
    double b_norm[1024];
    int32_t n_b;
    int32_t iters_used;
    double omega_last;
    int32_t n_indef;  /* PCG iterations with <z,r> <= 0 (r != 0) in the last frame */
    int32_t n_setups; /* setups run since creation */
    double setup_ms;  /* wall time of the setup in the last frame (0 if none; timing only, bench.py) */
};

static double wall_ms(void) {
    struct timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return 1e3 * (double)t.tv_sec + 1e-6 * (double)t.tv_nsec;
}

orc_sim* orc_sim_create(int kind, int32_t n_verts, int32_t m, const int32_t* verts,
                        const double* rest_pos, const double* pos, const double* vel,
                        const double* inv_mass, const double* compliance, const orc_config* cfg) {
    orc_sim* s = xcalloc(1, sizeof(orc_sim));
    s->kind = kind; s->n = n_verts; s->m = m; s->cfg = *cfg;
    size_t n3 = 3 * (size_t)n_verts;
    s->verts = xmalloc(sizeof(int32_t) * (size_t)m * kind);
    memcpy(s->verts, verts, sizeof(int32_t) * (size_t)m * kind);
    s->x = xmalloc(sizeof(double) * n3); s->v = xcalloc(n3, sizeof(double));
    s->x_old = xmalloc(sizeof(double) * n3); s->dx = xmalloc(sizeof(double) * n3);
    memcpy(s->x, pos ? pos : rest_pos, sizeof(double) * n3);
    if (vel) memcpy(s->v, vel, sizeof(double) * n3);
    s->w = xmalloc(sizeof(double) * (size_t)n_verts); memcpy(s->w, inv_mass, sizeof(double) * (size_t)n_verts);
    s->alpha = xmalloc(sizeof(double) * (size_t)m); memcpy(s->alpha, compliance, sizeof(double) * (size_t)m);
    if (kind == 2) {
        s->rest_len = xmalloc(sizeof(double) * (size_t)m);
        orc_rest_distance(m, verts, rest_pos, s->rest_len);
    } else {
        s->Dm_inv = xmalloc(sizeof(double) * 9 * (size_t)m);
        s->vol = xmalloc(sizeof(double) * (size_t)m);
        orc_rest_arap(m, verts, rest_pos, s->Dm_inv, s->vol);
    }
    s->C = xmalloc(sizeof(double) * (size_t)m);
    s->g = xmalloc(sizeof(double) * (size_t)m * kind * 3);
    s->lambda = xcalloc((size_t)m, sizeof(double));
    s->dl = xmalloc(sizeof(double) * (size_t)m);
    s->b = xmalloc(sizeof(double) * (size_t)m);
    s->atilde = xmalloc(sizeof(double) * (size_t)m);
    s->rowptr = xmalloc(sizeof(int64_t) * ((size_t)m + 1));
    s->nnz = orc_pattern(m, kind, verts, n_verts, s->rowptr, NULL);
    s->col = xmalloc(sizeof(int32_t) * (size_t)s->nnz);
    orc_pattern(m, kind, verts, n_verts, s->rowptr, s->col);
    s->val = xmalloc(sizeof(double) * (size_t)s->nnz);
    return s;
}

/* One frame (Algorithm 1).  Setup runs at ite 0 of frames with frame % setup_interval == 0, or
 * when marked stale (reading c13); Galerkin values are refreshed every iteration.
 * The outer break (l.12) is disabled: fixed n_iters (reading c11).  Collision (l.16) is out of
 * scope.  A PCG iteration with <z,r> <= 0 (the lazily-set omega of PAPER.md:320 no longer below
 * 2/lambda_max) is counted; with cfg.resetup_on_indef it marks the hierarchy stale, so setup re-runs
 * at ite 0 of the next frame (reading c13); without it the schedule is the literal
 * PAPER.md:215.  Returns 0, or -5 if a coarsest matrix is not SPD. */
int orc_sim_step(orc_sim* s, double dt, int32_t n_iters) {
    int rc = 0;
    s->n_indef = 0;
    s->setup_ms = 0.0;
    int32_t n = s->n, m = s->m;
    /* l.1 semiEuler: x_old = x; v += dt g (w > 0); x = x~ = x + dt v;  l.2 lambda = 0 */
    for (int32_t v = 0; v < n; ++v)
        for (int r = 0; r < 3; ++r) {
            int64_t k = 3 * (int64_t)v + r;
            s->x_old[k] = s->x[k];
            if (s->w[v] > 0.0) s->v[k] += dt * s->cfg.gravity[r];
            s->x[k] += dt * s->v[k];
        }
    for (int32_t j = 0; j < m; ++j) { s->lambda[j] = 0.0; s->atilde[j] = s->alpha[j] / (dt * dt); }
    s->n_b = 0;
    /* omega of l.11: user-specified, or halved whenever ||b|| rises (reading c21) */
    double omega = s->cfg.omega_relax, bprev = -1.0, b0 = 0.0;
    struct timespec tf0;
    clock_gettime(CLOCK_MONOTONIC, &tf0);
    for (int32_t ite = 0; ite < n_iters; ++ite) {
        if (s->kind == 2) orc_eval_distance(m, s->verts, s->x, s->rest_len, s->C, s->g);          /* l.4 */
        else orc_eval_arap(m, s->verts, s->x, s->Dm_inv, s->C, s->g);
        orc_assemble(m, s->kind, s->verts, s->w, s->g, s->atilde, s->rowptr, s->col, s->val);   /* l.5 */
        orc_rhs(m, s->C, s->atilde, s->lambda, s->b);                                            /* l.6 */
        const double bn = sqrt(dot(m, s->b, s->b));
        if (s->n_b < 1024) s->b_norm[s->n_b++] = bn;
        if (ite == 0) b0 = bn;
        if (s->cfg.backtrack && ite > 0 && bn > bprev) omega = fmax(0.5 * omega, s->cfg.omega_min);
        bprev = bn;
        if (ite == 0 && (s->h == NULL || s->stale || s->frame % s->cfg.setup_interval == 0)) { /* l.7 */
            const double t0 = wall_ms();
            orc_hier_free(s->h);
            s->h = orc_hier_build(m, s->rowptr, s->col, s->val, &s->cfg);
            s->stale = 0;
            s->n_setups++;
            s->setup_ms = wall_ms() - t0;
            if (factor_coarsest(s->h) != 0) rc = -5;
        } else {
            if (orc_hier_refresh(s->h, s->val) != 0) rc = -5;
            if (ite == 0 && s->cfg.omega_refresh_iters > 0) orc_hier_refresh_omega(s->h, s->cfg.omega_refresh_iters);
        }
        s->n_indef += orc_pcg(s->h, s->b, s->cfg.pcg_iters, s->dl, NULL);                         /* l.8 */
        orc_apply_dx(m, s->kind, s->verts, n, s->w, s->g, s->dl, s->dx);                         /* l.9 */
        for (int32_t j = 0; j < m; ++j) s->lambda[j] += s->dl[j];                               /* l.10 */
        for (int64_t k = 0; k < 3 * (int64_t)n; ++k) s->x[k] += omega * s->dx[k];              /* l.11 */
        s->iters_used = ite + 1;
        if (s->cfg.residual_tol > 0.0 && bn < s->cfg.residual_tol * b0) break;                 /* l.12 */
        if (s->cfg.residual_abs > 0.0 && bn < s->cfg.residual_abs) break;
        if (s->cfg.time_budget_ms > 0.0) {                                                       /* l.12 budget */
            struct timespec tn;
            clock_gettime(CLOCK_MONOTONIC, &tn);
            const double ms = (double)(tn.tv_sec - tf0.tv_sec) * 1e3 + (double)(tn.tv_nsec - tf0.tv_nsec) * 1e-6;
            if (ms > s->cfg.time_budget_ms) break;
        }
    }
    s->omega_last = omega;
    for (int64_t k = 0; k < 3 * (int64_t)n; ++k) s->v[k] = (s->x[k] - s->x_old[k]) / dt;      /* l.17 */
    s->frame++;
    if (s->n_indef && s->cfg.resetup_on_indef) s->stale = 1;
    return rc;
}

void orc_sim_mark_stale(orc_sim* s) { s->stale = 1; }
int32_t orc_sim_iters_used(const orc_sim* s) { return s->iters_used; }
double orc_sim_omega(const orc_sim* s) { return s->omega_last; }
int32_t orc_sim_indefinite_events(const orc_sim* s) { return s->n_indef; }
int32_t orc_sim_setups(const orc_sim* s) { return s->n_setups; }
double orc_sim_setup_ms(const orc_sim* s) { return s->setup_ms; }
void orc_sim_get(const orc_sim* s, double* x, double* v, double* lambda) {
    if (x) memcpy(x, s->x, sizeof(double) * 3 * (size_t)s->n);
    if (v) memcpy(v, s->v, sizeof(double) * 3 * (size_t)s->n);
    if (lambda) memcpy(lambda, s->lambda, sizeof(double) * (size_t)s->m);
}
void orc_sim_set(orc_sim* s, const double* x, const double* v) {
    if (x) memcpy(s->x, x, sizeof(double) * 3 * (size_t)s->n);
    if (v) memcpy(s->v, v, sizeof(double) * 3 * (size_t)s->n);
}
const orc_hier* orc_sim_hier(const orc_sim* s) { return s->h; }
int64_t orc_sim_nnz(const orc_sim* s) { return s->nnz; }
void orc_sim_get_A(const orc_sim* s, int64_t* rowptr, int32_t* col, double* val) {
    if (rowptr) memcpy(rowptr, s->rowptr, sizeof(int64_t) * ((size_t)s->m + 1));
    if (col) memcpy(col, s->col, sizeof(int32_t) * (size_t)s->nnz);
    if (val) memcpy(val, s->val, sizeof(double) * (size_t)s->nnz);
}
void orc_sim_get_b_norms(const orc_sim* s, double* out, int32_t n) {
    for (int32_t i = 0; i < n && i < s->n_b; ++i) out[i] = s->b_norm[i];
}
void orc_sim_free(orc_sim* s) {
    if (!s) return;
    orc_hier_free(s->h);
    free(s->verts); free(s->x); free(s->v); free(s->x_old); free(s->w); free(s->alpha);
    free(s->rest_len); free(s->Dm_inv); free(s->vol); free(s->C); free(s->g); free(s->lambda);
    free(s->dl); free(s->b); free(s->atilde); free(s->dx); free(s->rowptr); free(s->col); free(s->val);
    free(s);
}
