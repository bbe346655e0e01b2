// Matrix-free level-0 operator (PAPER.md:450 names it as future work).
//
// With the scaled gradients h_{i,s} = sqrt(w_v) grad_v C_i (v = verts[i][s]) the dual matrix of
// PAPER.md Eq. 4-5 is A = H H^T + diag(at), at_i = alpha_i / dt^2 (reading c14: the sum runs over every
// shared vertex).  A x is evaluated in two gathers instead of streaming the assembled CSR:
//   u_v     = sum_{(j,s): verts[j][s] = v} h_{j,s} x_j               (vertex gather, vertices [v0, v1))
//   (A x)_i = sum_s h_{i,s} . u_{verts[i][s]} + at_i x_i              (constraint gather, rows [row0, row1))
// followed by the same per-row epilogues as the CSR passes (PASS_* in solve.cuh).  The assembled CSR
// is still built every outer iteration: the Galerkin refresh (Eq. 6) and the smoother diagonal use it.
#pragma once
#include <functional>
#include <vector>

#include "common.cuh"

namespace mgpbd {

template <class T>
struct MatFree {
    int kc = 4;                     // vertices per constraint (2 distance, 4 tetrahedron)
    int32_t m = 0;                  // constraints
    int32_t row0 = 0, row1 = 0;     // constraint rows this rank evaluates
    int32_t v0 = 0, v1 = 0;         // vertices those rows touch
    const int32_t* verts = nullptr; // m x kc
    const T* h = nullptr;           // m x kc x 3
    const int64_t* vptr = nullptr;  // vertex incidence CSR (nv + 1)
    const int32_t* vlist = nullptr; // constraint*kc + slot, ascending per vertex
    int64_t ninc = 0;               // vptr[nv]
    int64_t e0 = 0, e1 = 0;         // vptr[v0], vptr[v1]
    // padded vertex-major layout of the hot gathers: vertex v's incidences (vlist order) start at ppos[v], a
    // multiple of 4, and are zero-padded to a multiple of 4, so every lane streams 16-byte vectors
    const int64_t* ppos = nullptr;  // nv + 1
    int64_t npad = 0;               // ppos[nv]
    int64_t p0 = 0, p1 = 0;         // ppos[v0], ppos[v1]
    const int32_t* vsrc = nullptr;  // npad: incidence code (constraint*kc + slot) of each padded slot, -1 = pad
    const uint16_t* vj16 = nullptr; // npad: constraint index - jbase[v] (when every vertex spans < 65536 rows)
    const int32_t* vj32 = nullptr;  // npad: constraint index (otherwise)
    const int32_t* jbase = nullptr; // nv
    T* hv = nullptr;                // vertex-major copy of h: [x | y | z] planes of npad values (padded layout)
    T* at = nullptr;                // alpha_i / dt^2 (m)
    T* u = nullptr;                 // 4 values per vertex (xyz, pad)
    const T* dinv = nullptr;        // 1 / A_ii from the assembly
    int grid = 1;                   // CTAs of the row kernel = number of dot partials
    bool tma = false;               // TMA-pipelined row kernel (persistent CTAs, bulk copies)
    int vg_grid_cap = 0;            // > 0: cap on the vertex-gather grid (MGPBD_MF_GRID_CAP, tests only)
    // != nullptr: the row kernel's last CTA also sums the dot partials (fixed order): JACOBI_DOT -> fin[0] (parts),
    // fin[1] (parts2); SPMV_DOT -> fin[2]; fin_ctr = arrival counter (0 between launches)
    int32_t vi0 = 0, vi1 = 0;       // interior vertices of a partitioned level 0 (no halo incidence), vi0 >= vi1: none
    bool vg_pdl = false;            // vertex gather launched with programmatic dependent launch (MGPBD_VG_PDL)
    double* fin = nullptr;
    unsigned* fin_ctr = nullptr;
    // TMA row kernel: vertex ids as 16-bit offsets from a per-tile base (tiles of the kernel's tiling from
    // row0 & ~3) when every tile spans < 65536 vertices; nullptr = the 32-bit verts
    const uint16_t* v16 = nullptr;  // m x kc
    const int32_t* vbase = nullptr; // per tile
    // TMA-pipelined vertex gather: slots per vertex tile (> 0 enables it) and its persistent grid
    int vg_ts = 0, vg_grid = 0;
};

// Plan of the TMA vertex gather over vertices [v0, v1) of the padded layout (host ppos): returns the stage
// capacity in slots (0: not usable) and the persistent grid in *grid.
int mf_vg_plan(const std::vector<int64_t>& ppos, int32_t v0, int32_t v1, int tsize, bool j16, int* grid);

// Build the 16-bit vertex-offset copy of verts (host copy hverts, m x kc) for the TMA tiling of rows
// [row0, row1).  Returns false (buffers untouched) if a tile spans >= 65536 vertices.
bool mf_build_v16(int32_t row0, int32_t row1, int kc, int tsize, const std::vector<int32_t>& hverts,
                  DBuf<uint16_t>& v16, DBuf<int32_t>& vbase, cudaStream_t s);

int mf_grid(int32_t rows);
// persistent grid of the TMA row kernel for rows [row0, row1) (T of tsize bytes, kc vertices)
int mf_grid_tma(int32_t row0, int32_t row1, int tsize, int kc, int vbytes = 4);


// Per outer iteration, after the constraint evaluation: hv (vertex-major h), at (all rows) and the
// diagonal inverse dinv of the owned rows.
template <class T>
void mf_refresh(const MatFree<T>& A, const double* alpha, double dt, T* dinv, cudaStream_t s);

// Eq. 5 from the vertex-major copy hv: x_v += omega sqrt(w_v) sum_{(j,s) at v} h_{j,s} dl_j
// for the vertices [v0, v1) (hv must be current: after mf_refresh of this outer iteration).
template <class T>
void mf_update(const MatFree<T>& A, const T* dl, const double* sqrtw, const double* omega, double* x, cudaStream_t s);

// One level-0 pass of `mode` (PASS_JACOBI, PASS_JACOBI_DOT, PASS_RESID_P, PASS_SPMV_DOT, PASS_POWER);
// same arguments and outputs as csr_pass, A.grid partials.
// x0_omega != 0 (PASS_JACOBI, TMA row kernel): x is not read — x_i = x0_omega D^-1_ii b_i, the first smoothing
// step from x = 0 fused into the second (the V-cycle's k_jacobi0 expression, bit for bit).
template <class T>
// mid != nullptr (partitioned level 0): called between the gather of the interior vertices [vi0, vi1) and the
// boundary vertices — the caller joins the halo exchange there, which therefore overlaps the interior gather.
void mf_pass(int mode, const MatFree<T>& A, const T* x, const T* b, T* y, const T* aux, double omega,
             double* parts, double* parts2, cudaStream_t s, double alpha = 0.0, const T* xprev = nullptr,
             double x0_omega = 0.0, const std::function<void()>* mid = nullptr);

}  // namespace mgpbd
