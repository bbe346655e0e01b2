// Host orchestration of one MGPBD frame (Algorithm 1) and the extern "C" ABI of mgpbd.h.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/mgpbd.h"
#include "common.cuh"
#include "mesh.cuh"
#include "setup.cuh"
#include "solve.cuh"
#include "util.cuh"
#include "comm.cuh"
#include "matfree.cuh"
#include "vagal.cuh"
#include "coarse.cuh"
#include "coarse_res.cuh"
#include "nullspace.cuh"
#include "coarse_tail.cuh"
#include "subcycle.cuh"

namespace mgpbd {

static int choose_vl(int64_t n, int64_t nnz) {
    double avg = n ? (double)nnz / (double)n : 1.0;
    int vl = 2;
    while (vl < 32 && vl * 1.5 < avg) vl *= 2;
    return vl < 4 ? 4 : vl;
}

struct EngineBase {
    virtual ~EngineBase() = default;
    virtual void step(double dt, int32_t n_iters) = 0;
    virtual void set_state(const double* pos, const double* vel) = 0;
    virtual void get_positions(double* out) = 0;
    virtual void get_velocities(double* out) = 0;
    virtual void get_lambda(double* out) = 0;
    virtual void get_stats(mgpbd_stats* st) = 0;
    virtual void level_sizes(int l, int64_t* n, int64_t* nnz) = 0;
    virtual void get_level(int l, int64_t* rowptr, int32_t* col, double* val) = 0;
    virtual void get_prolongator(int l, double* p) = 0;
    virtual void get_prolongator_csr(int l, int64_t* nnz, int64_t* rowptr, int32_t* col, double* val) = 0;
    virtual void get_aggregates(int l, int32_t* a) = 0;
    virtual void get_near_kernel(double* b) = 0;
    virtual void debug_setup_from(const double* vals) = 0;
    virtual void debug_vcycle(const double* b, double* x) = 0;
    virtual void debug_pcg(const double* b, int32_t iters, double* x) = 0;
    virtual void debug_prepare(double dt) = 0;
    virtual void pass_burst(int32_t reps, double* ms, double* bytes) = 0;
    virtual void bind() = 0;  // make this context's device/stream current for the calling thread
    virtual void set_profiling(int on) = 0;
    bool stale = true;
};

template <class T>
class Engine : public EngineBase {
   public:
    struct Level {
        int32_t n = 0;
        int64_t nnz = 0;
        DBuf<int64_t> rowptr_own;
        DBuf<int32_t> col_own;
        const int64_t* rowptr = nullptr;
        const int32_t* col = nullptr;
        DBuf<T> val, dinv;            // hot values
        DBuf<double> val64, dinv64;   // setup values
        // towards level+1
        DBuf<int32_t> agg;
        int32_t n_agg = 0;
        DBuf<double> P64;
        DBuf<T> P;
        DBuf<int64_t> mptr;
        DBuf<int32_t> mlist;
        GalerkinPlan plan;
        DBuf<T> tval;
        DBuf<double> tval64;
        double omega = 0.0;
        double sm_omega[8] = {0, 0, 0, 0, 0, 0, 0, 0}, sm_alpha[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // set_smoother
        // multicolour GS smoother (smoother = 2): rows grouped by colour
        DBuf<int64_t> gs_ptr;
        DBuf<int32_t> gs_list;
        int gs_ncol = 0;
        // V-cycle vectors
        DBuf<T> vb, vz, vx, vy, vt;
        int vl = 32, grid = 1, vlr = 0, tile_nnz = 0;
        int band_rows = 0, band_grid = 0, prod_cap = 0, band_win = 0, row_vl = 0;
        DBuf<int32_t> win_lo, win_len;
        DBuf<uint16_t> col16;
        // rows this rank processes in the hot loop (partitioned level 0); coarse levels: all rows
        int32_t own0 = 0, own1 = -1;
        int32_t own_n() const { return (own1 < 0 ? n : own1) - own0; }
        // k > 1 near kernel (f2, nullspace.cuh): general prolongator towards level+1 and the block Galerkin
        int kk = 1;
        KProlongator kp;
        DBuf<T> kQs, kpval, kW, kones;
        DBuf<double> kW64;
        DBuf<int64_t> arow, xoff;   // aggregate-level coarse pattern (rows), block offsets per entry
        DBuf<double> pwv;           // last normalised power iterate (start of the omega refresh, c26)
        DBuf<int32_t> acol, erow;
        void configure(cudaStream_t s) {
            const int32_t nl = own_n();
            vl = choose_vl(n, nnz);
            tile_config(n, nnz, rowptr, vlr, grid, tile_nnz, s);  // full-range tiling (replicated setup)
            if (nl != n) {  // the owned range is tiled from own0: size shared memory for both tilings
                int vlr2 = 0, grid2 = 0, tn2 = 0;
                tile_config(nl, nnz, rowptr + own0, vlr2, grid2, tn2, s);
                tile_nnz = std::max(tile_nnz, tn2);
                if (vlr2 == 0 || tile_nnz * 8 > 200 * 1024) vlr = 0;
            }
            if (vlr == 0) grid = pass_grid(n, vl);
            band_rows = 0;
            if (!std::getenv("MGPBD_NO_BAND"))
                band_config<T>(own0, nl, rowptr, col, vlr, win_lo, win_len, band_rows, band_grid, prod_cap, band_win,
                               row_vl, col16, s);
        }
        // hot == true: this rank's rows with the band kernels; false: all rows (replicated setup)
        template <class U>
        Csr<U> view(const U* v, const U* d, bool hot_rows) const {
            Csr<U> c;
            c.row0 = hot_rows ? own0 : 0;
            c.n = hot_rows ? own_n() : n;
            c.nnz = nnz; c.rowptr = rowptr; c.col = col; c.val = v; c.dinv = d;
            c.vl = vl; c.grid = grid; c.vlr = vlr; c.tile_nnz = tile_nnz;
            c.nparts = grid;
            if (hot_rows && band_rows) {
                c.band_rows = band_rows; c.band_grid = band_grid; c.prod_cap = prod_cap; c.band_win = band_win;
                c.row_vl = row_vl;
                c.col16 = col16.p;
                c.win_lo = win_lo.p; c.win_len = win_len.p;
                c.nparts = band_grid;
            }
            return c;
        }
        Csr<T> hot() const { return view<T>(val.p, dinv.p, true); }
        Csr<double> setup_csr() const { return view<double>(val64.p, dinv64.p, false); }
    };

    mgpbd_config cfg;
    cudaStream_t st = nullptr;
    bool own_stream = false;
    int kind = 2, kc = 2;
    int kk = 1;  // near-kernel vectors per aggregate (cfg.k_nullspace)
    int32_t nv = 0, m = 0;
    DBuf<int32_t> verts;
    DBuf<double> x, v, x_old, w, sqrtw, alpha, rest, vol, lambda;
    DBuf<int64_t> vptr, rowptr0;
    DBuf<int32_t> vlist, col0;
    int64_t nnz0 = 0;
    DBuf<T> h, b0;
    DBuf<double> h64, b64, at64;
    std::vector<std::unique_ptr<Level>> L;
    int nL = 0;
    bool have_hier = false;
    DBuf<double> Ainv, inv_work;
    DBuf<T> r, p, q, xs;
    DBuf<double> scal, parts1, parts2, bn, B0, pw_v, pw_w, pw_ss, mf_fin;
    DBuf<unsigned> mf_fin_ctr;
    DBuf<int> flags;
    int32_t ncolours = 0;
    int64_t frame = 0;
    int setup_ran = 0;
    int n_b = 0;
    double ms_setup = 0, ms_frame = 0;
    // profiling of the level-0 matrix passes
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    double l0_ms = 0, l0_bytes = 0;
    int64_t l0_launches = 0;
    double l0_bytes_acc = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_pairs;
    // phase times of the last frame (profile = 1, eager launches): assemble, Galerkin refresh, V-cycle,
    // whole MGPCG, update
    enum { PH_ASM, PH_GAL, PH_VC, PH_PCG, PH_UPD, PH_N };
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ph_pairs[PH_N];
    double ph_ms[PH_N] = {0, 0, 0, 0, 0};
    template <class F>
    void timed(int ph, F&& f) {
        if (!cfg.profile || capturing) { f(); return; }
        cudaEvent_t e0 = ev();
        MG_CK(cudaEventRecord(e0, st));
        f();
        cudaEvent_t e1 = ev();
        MG_CK(cudaEventRecord(e1, st));
        ph_pairs[ph].emplace_back(e0, e1);
    }
    int64_t launches_last = 0;
    int32_t indef_events = 0;
    // partitioned level 0 (world > 1): rows [r0, r1) of this rank, halo transfers
    std::unique_ptr<Comm> comm;
    bool dist = false;
    int32_t r0 = 0, r1 = 0;
    int64_t nnz_own = 0, halo_elems = 0;
    std::vector<Comm::Xfer> xfers;
    std::vector<int32_t> part_bounds;  // level-0 row blocks of all ranks
    int64_t tb0 = 0, te0 = -1;  // Galerkin segments of the owned rows (level 0 -> 1)
    DBuf<double> dsc;           // rank-local dot results before the allreduce
    // matrix-free level-0 operator (cfg.level0_operator == 1, matfree.cuh)
    MatFree<T> mf;
    DBuf<T> mf_hv, mf_at, mf_u;
    // padded vertex-major layout shared by mf and mf64 (matfree.cuh)
    DBuf<int64_t> mf_ppos;
    DBuf<int32_t> mf_vsrc, mf_vj32, mf_jbase;
    DBuf<uint16_t> mf_vj16, mf_v16, mf64_v16;
    DBuf<int32_t> mf_vbase, mf64_vbase;
    int64_t mf_npad = 0;
    // fp64 matrix-free operator for the setup's level-0 power method (reading c18: setup in fp64)
    MatFree<double> mf64;
    DBuf<double> mf64_hv, mf64_at, mf64_u;
    bool mf64_ok = false;
    // Jones-Plassmann colouring of A_0's pattern (reading c5): depends only on the fixed pattern
    DBuf<int32_t> colours0;
    bool colours_cached = false;
    bool mf_ready = false;      // h is current and describes level 0 (false after debug_setup_from)
    VaPlan va;                  // level-0 -> 1 Galerkin from h (vagal.cuh), rebuilt at every setup
    bool va_ok = false;
    int64_t omega_refreshes = 0;
    bool eval_hv = std::getenv("MGPBD_NO_EVAL_HV") == nullptr;  // evaluation writes the vertex-major operator data
    DBuf<int32_t> mf_inv;
    bool npad_fits() const { return mf_npad < ((int64_t)1 << 31); }
    // halo exchange overlapped with the interior vertex gather (partitioned matrix-free level 0; MGPBD_NO_HALO_OVERLAP)
    bool halo_overlap = std::getenv("MGPBD_NO_HALO_OVERLAP") == nullptr;
    cudaStream_t st_comm = nullptr;
    cudaEvent_t ev_xa = nullptr, ev_xb = nullptr;
    // level-0 x1 of the next V-cycle already formed by the PCG x / r update (one launch less per iteration)
    bool l0_x1_ready = false;
    bool vc_trace = false;  // stage stamps inside the first level-0 V-cycle of an iteration (MGPBD_TRACE_STAGES)
    // the row kernel's last CTA sums the PCG dot partials (MatFree::fin) on this path
    const double* fin_ready() const {
        return (!dist && nL > 1 && mf_on() && mf.tma && mf.fin && cfg.smoother != 2) ? mf.fin : nullptr;
    }
    bool x1_fusable() const {
        return !dist && nL > 1 && cfg.smoother != 2 && !fuse_jacobi0 && std::getenv("MGPBD_NO_X1_FUSE") == nullptr;
    }
    // dense bottom of the cycle (reading c27; MGPBD_DENSE_CUT = max rows, 0 = off)
    int dense_cut = std::getenv("MGPBD_DENSE_CUT") ? std::atoi(std::getenv("MGPBD_DENSE_CUT")) : 1024;
    int lcut = -1;
    bool sub_ok = false;
    SubCycle<T> subc;
    DBuf<double> Mcut;
    bool va_setup0 = false;  // the last setup formed level 1 through the VA plan (fp64 omega refresh follows it)
    bool va_off = std::getenv("MGPBD_NO_VA_SETUP") != nullptr;  // CSR Galerkin at setup (comparison)
    double last_dt = 0.0;
    DBuf<double> omega_dev;     // relaxation omega of Alg. 1 l.11 (device scalar: backtracking, c21)
    double omega_last = 0.0;
    // levels >= 1 of the V-cycle as one persistent kernel (coarse.cuh); MGPBD_NO_COARSE_KERNEL=1 disables
    CoarseCycle<T> ccyc;
    bool ccyc_ok = false;
    bool use_coarse_kernel = std::getenv("MGPBD_NO_COARSE_KERNEL") == nullptr;
    DBuf<unsigned long long> ctrace;
    // shared-memory-resident variant of the coarse kernel (coarse_res.cuh); MGPBD_NO_RES_COARSE=1 disables
    ResPlan res_plan;
    DBuf<ResLevel> res_lv;
    DBuf<ResCopy> res_cp;
    DBuf<int32_t> res_nc;
    DBuf<uint32_t> res_tx;
    bool res_ok = false;
    bool use_res = std::getenv("MGPBD_NO_RES_COARSE") == nullptr;
    // smallest levels on one thread-block cluster (coarse_tail.cuh); the levels above it run as the down /
    // up halves of the resident kernel over a truncated cycle.  MGPBD_NO_TAIL=1 disables
    TailPlan tail;
    bool tail_ok = false;
    bool use_tail = std::getenv("MGPBD_NO_TAIL") == nullptr;
    // the V-cycle's first two level-0 smoothing steps as one pass (MGPBD_FUSE_J0=1): measured 1.2 ms/frame
    // SLOWER in the bench (the vertex gather then gathers D^-1 and b instead of x), so off by default
    bool fuse_jacobi0 = std::getenv("MGPBD_FUSE_J0") != nullptr;
    CoarseCycle<T> ccyc_top;
    ResPlan res_top;
    // fused variant: ONE cooperative launch with cluster dimensions runs the grid down half, the tail on its
    // first cluster and the up half (no kernel boundaries); MGPBD_NO_FUSED_TAIL=1 keeps the three launches
    TailPlan tail_f;
    bool fused_ok = false;
    bool use_fused = std::getenv("MGPBD_NO_FUSED_TAIL") == nullptr;
    CoarseCycle<T> ccyc_f;
    ResPlan res_f;
    TailArgs<T> targs_f;
    uint32_t tail_base_f = 0;
    DBuf<ResLevel> rf_lv;
    DBuf<ResCopy> rf_cp;
    DBuf<int32_t> rf_nc;
    DBuf<uint32_t> rf_tx;
    DBuf<ResLevel> rt_lv;
    DBuf<ResCopy> rt_cp;
    DBuf<int32_t> rt_nc;
    DBuf<uint32_t> rt_tx;
    int ccyc_from = std::getenv("MGPBD_COARSE_FROM") ? std::atoi(std::getenv("MGPBD_COARSE_FROM")) : 1;
    bool mf_on() const { return cfg.level0_operator == 1 && mf_ready; }

    void setup_partition() {
        if (cfg.vgroup) comm = make_virtual_comm(static_cast<VirtualGroup*>(cfg.vgroup), cfg.rank);
        else comm = make_nccl_comm(cfg.nccl_id, cfg.rank, cfg.world, cfg.device);
        dist = true;
        const int W = cfg.world, me = cfg.rank;
        std::vector<int64_t> hrp((size_t)m + 1);
        d2h(hrp.data(), rowptr0.p, (size_t)m + 1, st);
        MG_CK(cudaStreamSynchronize(st));
        const std::vector<int32_t> bounds = partition_rows(hrp.data(), m, W);
        part_bounds = bounds;
        std::vector<int32_t> mn(W), mx(W);
        for (int q = 0; q < W; ++q) row_range_window(rowptr0.p, col0.p, bounds[q], bounds[q + 1], &mn[q], &mx[q], st);
        const auto plan = halo_plan(bounds, mn, mx);
        r0 = bounds[me];
        r1 = bounds[me + 1];
        nnz_own = hrp[r1] - hrp[r0];
        xfers.clear();
        halo_elems = 0;
        for (int p = 0; p < W; ++p) {
            if (p == me) continue;
            Comm::Xfer x{p, plan[p][me], plan[me][p]};
            if (x.send.size() || x.recv.size()) xfers.push_back(x);
            halo_elems += x.recv.size();
        }
        dsc.resize(4);
    }
    // Padded vertex-major incidence layout of the hot vertex gather (matfree.cuh): vertex v's incidences
    // (vlist order) at ppos[v] .. ppos[v] + deg(v), zero-padded to a multiple of 4; constraint indices as
    // 16-bit offsets from the vertex's smallest one when every vertex spans < 65536 constraints.
    std::vector<int64_t> ppos_h;
    void build_padded_layout(const std::vector<int64_t>& hp) {
        const int64_t ninc = hp[nv];
        std::vector<int32_t> vl((size_t)ninc);
        d2h(vl.data(), vlist.p, (size_t)ninc, st);
        MG_CK(cudaStreamSynchronize(st));
        ppos_h.assign((size_t)nv + 1, 0);
        for (int32_t v = 0; v < nv; ++v) ppos_h[v + 1] = ppos_h[v] + ((hp[v + 1] - hp[v] + 3) & ~(int64_t)3);
        mf_npad = ppos_h[nv];
        std::vector<int32_t> src((size_t)mf_npad, -1), jb((size_t)nv, 0), j32((size_t)mf_npad, 0);
        bool fits16 = true;
        for (int32_t v = 0; v < nv; ++v) {
            int32_t jmin = INT32_MAX, jmax = -1;
            for (int64_t e = hp[v]; e < hp[v + 1]; ++e) {
                const int32_t j = vl[e] / kc;
                jmin = std::min(jmin, j); jmax = std::max(jmax, j);
                src[ppos_h[v] + (e - hp[v])] = vl[e];
                j32[ppos_h[v] + (e - hp[v])] = j;
            }
            jb[v] = jmax < 0 ? 0 : jmin;
            if (jmax >= 0 && jmax - jmin >= 65536) fits16 = false;
            for (int64_t p = ppos_h[v] + (hp[v + 1] - hp[v]); p < ppos_h[v + 1]; ++p) j32[p] = jb[v];  // pads: x[jbase]
        }
        if (std::getenv("MGPBD_NO_VJ16")) fits16 = false;
        mf_ppos.resize((size_t)nv + 1); h2d(mf_ppos.p, ppos_h.data(), (size_t)nv + 1, st);
        mf_vsrc.resize((size_t)mf_npad); h2d(mf_vsrc.p, src.data(), (size_t)mf_npad, st);
        {   // padded slot of every incidence code (constraint j, slot k) -> j kc + k: the evaluation writes hv directly
            std::vector<int32_t> inv((size_t)ninc, 0);
            for (int64_t p = 0; p < mf_npad; ++p)
                if (src[p] >= 0) inv[src[p]] = (int32_t)p;
            mf_inv.resize((size_t)ninc); h2d(mf_inv.p, inv.data(), (size_t)ninc, st);
        }
        mf_jbase.resize((size_t)nv); h2d(mf_jbase.p, jb.data(), (size_t)nv, st);
        if (fits16) {
            std::vector<uint16_t> j16((size_t)mf_npad);
            for (int32_t v = 0; v < nv; ++v)
                for (int64_t p = ppos_h[v]; p < ppos_h[v + 1]; ++p) j16[p] = (uint16_t)(j32[p] - jb[v]);
            mf_vj16.resize((size_t)mf_npad); h2d(mf_vj16.p, j16.data(), (size_t)mf_npad, st);
            mf_vj32.free_all();
        } else {
            mf_vj32.resize((size_t)mf_npad); h2d(mf_vj32.p, j32.data(), (size_t)mf_npad, st);
            mf_vj16.free_all();
            std::vector<int32_t> zero((size_t)nv, 0);
            h2d(mf_jbase.p, zero.data(), (size_t)nv, st);   // absolute indices
        }
        MG_CK(cudaStreamSynchronize(st));
    }

    void setup_matfree() {
        // vertices touched by this rank's rows: their incidences reference only owned or halo rows
        std::vector<int32_t> hv_((size_t)(r1 - r0) * kc);
        if (r1 > r0) d2h(hv_.data(), verts.p + (size_t)r0 * kc, hv_.size(), st);
        std::vector<int64_t> hp((size_t)nv + 1);
        d2h(hp.data(), vptr.p, (size_t)nv + 1, st);
        MG_CK(cudaStreamSynchronize(st));
        int32_t vmin = nv, vmax = -1;
        for (int32_t q : hv_) { vmin = std::min(vmin, q); vmax = std::max(vmax, q); }
        mf = MatFree<T>();
        mf.kc = kc;
        mf.m = m;
        mf.row0 = r0; mf.row1 = r1;
        mf.v0 = vmax < 0 ? 0 : vmin; mf.v1 = vmax < 0 ? 0 : vmax + 1;
        mf.verts = verts.p; mf.h = h.p; mf.vptr = vptr.p; mf.vlist = vlist.p;
        mf.ninc = hp[nv]; mf.e0 = hp[mf.v0]; mf.e1 = hp[mf.v1];
        build_padded_layout(hp);
        mf.ppos = mf_ppos.p; mf.npad = mf_npad; mf.vsrc = mf_vsrc.p; mf.jbase = mf_jbase.p;
        mf.vj16 = mf_vj16.n ? mf_vj16.p : nullptr; mf.vj32 = mf_vj32.n ? mf_vj32.p : nullptr;
        mf.p0 = ppos_h[mf.v0]; mf.p1 = ppos_h[mf.v1];
        if (dist && mf.v1 > mf.v0) {  // longest run of vertices whose incidences are all owned rows [r0, r1)
            std::vector<int32_t> vl_((size_t)hp[nv]);
            d2h(vl_.data(), vlist.p, vl_.size(), st);
            MG_CK(cudaStreamSynchronize(st));
            int32_t best0 = 0, best1 = 0, run0 = -1;
            for (int32_t v = mf.v0; v <= mf.v1; ++v) {
                bool interior = v < mf.v1;
                for (int64_t e = v < mf.v1 ? hp[v] : 0; interior && e < hp[v + 1]; ++e) {
                    const int32_t j = vl_[e] / kc;
                    interior = j >= r0 && j < r1;
                }
                if (interior && run0 < 0) run0 = v;
                if (!interior && run0 >= 0) {
                    if (v - run0 > best1 - best0) { best0 = run0; best1 = v; }
                    run0 = -1;
                }
            }
            mf.vi0 = best0; mf.vi1 = best1;
        }
        mf_hv.resize(3 * (size_t)mf_npad); mf_at.resize(m); mf_u.resize(4 * (size_t)nv);
        MG_CK(cudaMemsetAsync(mf_hv.p, 0, sizeof(T) * 3 * (size_t)mf_npad, st));  // pad slots stay 0 (EvalHv)
        MG_CK(cudaMemsetAsync(mf_u.p, 0, sizeof(T) * 4 * (size_t)nv, st));
        mf.hv = mf_hv.p; mf.at = mf_at.p; mf.u = mf_u.p;
        mf.dinv = L[0]->dinv.p;
        if (!dist) {  // fp64 twin on the same geometry (h64 / dinv64 of the setup assembly)
            mf64 = MatFree<double>();
            mf64.kc = kc; mf64.m = m; mf64.row0 = 0; mf64.row1 = m; mf64.v0 = 0; mf64.v1 = nv;
            mf64.verts = verts.p; mf64.vptr = vptr.p; mf64.vlist = vlist.p;
            mf64.ninc = hp[nv]; mf64.e0 = 0; mf64.e1 = hp[nv];
            mf64.ppos = mf_ppos.p; mf64.npad = mf_npad; mf64.vsrc = mf_vsrc.p; mf64.jbase = mf_jbase.p;
            mf64.vj16 = mf.vj16; mf64.vj32 = mf.vj32;
            mf64.p0 = 0; mf64.p1 = mf_npad;
            mf64_hv.resize(3 * (size_t)mf_npad); mf64_at.resize(m); mf64_u.resize(4 * (size_t)nv);
            MG_CK(cudaMemsetAsync(mf64_u.p, 0, sizeof(double) * 4 * (size_t)nv, st));
            mf64.hv = mf64_hv.p; mf64.at = mf64_at.p; mf64.u = mf64_u.p;
            mf64.tma = std::getenv("MGPBD_NO_TMA") == nullptr;
            mf64.grid = mf64.tma ? mf_grid_tma(0, m, 8, kc) : mf_grid(m);
            mf64_ok = true;
        }
        mf.tma = std::getenv("MGPBD_NO_TMA") == nullptr;
        mf.vg_pdl = std::getenv("MGPBD_NO_VG_PDL") == nullptr;  // 94.77 -> 94.64 ms/frame (tools/ab_frames.py)
        int vbytes = 4;
        if (mf.tma && !std::getenv("MGPBD_NO_V16")) {  // 16-bit vertex offsets per TMA tile (8 B per row saved)
            std::vector<int32_t> hvt((size_t)m * kc);
            d2h(hvt.data(), verts.p, hvt.size(), st);
            MG_CK(cudaStreamSynchronize(st));
            if (mf_build_v16(r0, r1, kc, (int)sizeof(T), hvt, mf_v16, mf_vbase, st)) {
                mf.v16 = mf_v16.p; mf.vbase = mf_vbase.p;
                vbytes = 2;
                // the fp64 twin (one rank: r0 = 0) has its own tiling when its tile height differs (cloth)
                if (mf64_ok && mf_build_v16(0, m, kc, 8, hvt, mf64_v16, mf64_vbase, st)) {
                    mf64.v16 = mf64_v16.p; mf64.vbase = mf64_vbase.p;
                }
            }
        }
        if (mf64_ok && mf64.tma) mf64.grid = mf_grid_tma(0, m, 8, kc, mf64.v16 ? 2 : 4);
        if (mf.tma && std::getenv("MGPBD_VG_TMA")) {  // TMA-pipelined vertex gather (measured slower in fp32: off)
            mf.vg_ts = mf_vg_plan(ppos_h, mf.v0, mf.v1, (int)sizeof(T), mf.vj16 != nullptr, &mf.vg_grid);
            if (mf64_ok) mf64.vg_ts = mf_vg_plan(ppos_h, 0, nv, 8, mf.vj16 != nullptr, &mf64.vg_grid);
        }
        mf.grid = mf.tma ? mf_grid_tma(r0, r1, (int)sizeof(T), kc, vbytes) : mf_grid(r1 - r0);
        if (const char* cap = std::getenv("MGPBD_MF_GRID_CAP")) {  // tests: many tiles per CTA (TMA ring wraps)
            const int c = std::max(1, std::atoi(cap));
            mf.grid = std::min(mf.grid, c);
            mf.vg_grid_cap = c;
            if (mf64_ok) { mf64.grid = std::min(mf64.grid, c); mf64.vg_grid_cap = c; }
        }
        // opt-in (MGPBD_FIN_IN_ROWS=1): the row kernel's last CTA sums the PCG dot partials; measured 0.2 ms/frame
        // slower (the arrival atomics lengthen every dot pass) than the redundant per-CTA sums of the update kernels
        if (mf.tma && !dist && std::getenv("MGPBD_FIN_IN_ROWS") != nullptr) {
            mf_fin.resize(4);
            mf_fin_ctr.resize(1);
            MG_CK(cudaMemsetAsync(mf_fin_ctr.p, 0, sizeof(unsigned), st));
            mf.fin = mf_fin.p;
            mf.fin_ctr = mf_fin_ctr.p;
        }

    }
    int l0_nparts() const { return mf_on() ? mf.grid : L[0]->hot().nparts; }

    int32_t lo0(int l) const { return (l == 0) ? r0 : 0; }
    int32_t cnt(int l) const { return (l == 0) ? r1 - r0 : L[l]->n; }

    Engine(const mgpbd_mesh* mesh, const mgpbd_constraints* cons, const double* inv_mass, const double* comp,
           const mgpbd_config* c) {
        cfg = *c;
        kk = cfg.k_nullspace;
        MG_CK(cudaSetDevice(cfg.device));
        if (cfg.stream) st = (cudaStream_t)cfg.stream;
        else { MG_CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)); own_stream = true; }
        // stream-ordered allocations from the default pool, retained across setups
        cudaMemPool_t pool;
        MG_CK(cudaDeviceGetDefaultMemPool(&pool, cfg.device));
        uint64_t keep = UINT64_MAX;
        MG_CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        g_alloc_stream = st;
        kind = cons->kind; kc = (int)kind;
        nv = mesh->n_verts; m = cons->n_cons;
        verts.resize((size_t)m * kc);
        h2d(verts.p, cons->verts, (size_t)m * kc, st);
        size_t n3 = 3 * (size_t)nv;
        x.resize(n3); v.resize(n3); x_old.resize(n3); w.resize(nv); sqrtw.resize(nv);
        DBuf<double> X;
        X.resize(n3);
        h2d(X.p, mesh->rest_pos, n3, st);
        h2d(x.p, mesh->pos ? mesh->pos : mesh->rest_pos, n3, st);
        if (mesh->vel) h2d(v.p, mesh->vel, n3, st);
        else MG_CK(cudaMemsetAsync(v.p, 0, n3 * sizeof(double), st));
        h2d(w.p, inv_mass, nv, st);
        sqrt_vec(nv, w.p, sqrtw.p, st);
        alpha.resize(m);
        h2d(alpha.p, comp, m, st);
        lambda.resize(m);
        MG_CK(cudaMemsetAsync(lambda.p, 0, sizeof(double) * (m ? m : 1), st));
        if (kind == 2) {
            rest.resize(m);
            rest_distance(verts.p, X.p, m, rest.p, st);
        } else {
            rest.resize(9 * (size_t)m); vol.resize(m);
            DBuf<int32_t> bad;
            bad.resize(1);
            MG_CK(cudaMemsetAsync(bad.p, 0, sizeof(int32_t), st));
            rest_arap(verts.p, X.p, m, rest.p, vol.p, bad.p, st);
            if (read_scalar(bad.p, st)) throw Error(MGPBD_E_ARG, "degenerate rest tetrahedron");
        }
        build_incidence(verts.p, m, kc, nv, vptr, vlist, st);
        build_pattern(verts.p, m, kc, nv, vptr.p, vlist.p, rowptr0, col0, st);
        nnz0 = read_scalar(rowptr0.p + m, st);
        r0 = 0; r1 = m; nnz_own = nnz0;
        if (cfg.world > 1 || cfg.vgroup || cfg.nccl_id) setup_partition();
        h.resize((size_t)m * kc * 3); b0.resize(m);
        r.resize(m); p.resize(m); q.resize(m); xs.resize(m);
        scal.resize(2 * 4096); flags.resize(8); bn.resize(MGPBD_MAX_FRAME_ITERS);
        parts1.resize(148 * 8); parts2.resize(148 * 8);
        pw_ss.resize(4);
        MG_CK(cudaMemsetAsync(flags.p, 0, 8 * sizeof(int), st));
        // level 0 skeleton (pattern fixed for the context's lifetime)
        L.clear();
        L.emplace_back(new Level());
        Level& l0 = *L[0];
        l0.n = m; l0.nnz = nnz0; l0.rowptr = rowptr0.p; l0.col = col0.p;
        l0.val.resize(nnz0); l0.dinv.resize(m);
        l0.own0 = r0; l0.own1 = r1;
        l0.configure(st);
        alloc_vectors(l0);
        MG_CK(cudaMemsetAsync(l0.vt.p, 0, sizeof(T) * m, st));  // restriction input: zero outside the owned rows
        if (cfg.level0_operator == 1) setup_matfree();
        if (use_graphs && dist && !comm->graph_capturable()) use_graphs = false;
        MG_CK(cudaStreamSynchronize(st));
    }

    ~Engine() override {
        invalidate_graphs();
        for (auto e : ev_pool) cudaEventDestroy(e);
        cudaStreamSynchronize(st);
        if (st_comm) { cudaStreamSynchronize(st_comm); cudaStreamDestroy(st_comm); }
        if (ev_xa) cudaEventDestroy(ev_xa);
        if (ev_xb) cudaEventDestroy(ev_xb);
        g_alloc_stream = nullptr;  // members are freed after this body: plain cudaFree from here on
        if (own_stream && st) cudaStreamDestroy(st);
    }
    void bind() override { cudaSetDevice(cfg.device); g_alloc_stream = st; }

    void alloc_vectors(Level& lv) {
        lv.vb.resize(lv.n); lv.vz.resize(lv.n); lv.vx.resize(lv.n); lv.vy.resize(lv.n); lv.vt.resize(lv.n);
    }

    cudaEvent_t ev() {
        if (ev_used == ev_pool.size()) {
            cudaEvent_t e;
            MG_CK(cudaEventCreate(&e));
            ev_pool.push_back(e);
        }
        return ev_pool[ev_used++];
    }

    // Algorithmic bytes of one level-0 CSR pass (matrix stream + per-row vectors), see DESIGN.md.
    double pass_bytes(int mode) const {
        const double s = sizeof(T);
        const double cb = (L[0]->band_rows > 0 && L[0]->row_vl > 0) ? 2.0 : 4.0;  // col16 hot copy or int32
        const double mrows = (double)(r1 - r0);
        double mat = (double)nnz_own * (s + cb) + 8.0 * (mrows + 1);
        if (mf_on()) {
            // matrix-free: vertex gather (hv planes, vlist, vptr, u write) + row gather (verts, h, at,
            // u read once per vertex); x is read by both kernels
            // padded slots: 3 planes + the 16/32-bit constraint index; per vertex ppos, jbase, u
            const double nvr = (double)(mf.v1 - mf.v0), np = (double)(mf.p1 - mf.p0);
            const double jb = mf.vj16 ? 2.0 : 4.0;
            mat = np * (3 * s + jb) + 8.0 * (nvr + 1) + (mf.vj16 ? 4.0 * nvr : 0.0) + nvr * 4 * s   // gather
                  + mrows * ((mf.v16 ? 2.0 : 4.0) * kc + 3.0 * kc * s + s) + nvr * 4 * s + mrows * s;  // rows
        }
        double vec;
        switch (mode) {
            case PASS_JACOBI: vec = 4 * s; break;          // x (gathered once), b, dinv, y
            case PASS_JACOBI_DOT: vec = 5 * s; break;      // + r
            case PASS_RESID_P: vec = 4 * s; break;         // x, b, P, t
            case PASS_SPMV_DOT: vec = 2 * s; break;        // x, y
            default: vec = 3 * s; break;
        }
        return mat + vec * mrows;
    }

    // ---- CUDA graphs: the solve part of each outer iteration (Galerkin refresh, coarsest inverse,
    // MGPCG, update) is captured once per hierarchy and replayed; graph i owns its profiling events.
    struct IterGraph {
        cudaGraphExec_t exec = nullptr;
        bool seen = false;  // first use runs eagerly (kernel attributes are set outside capture)
        std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
        int64_t launches = 0, l0_launches = 0;
        double l0_bytes = 0;
    };
    std::vector<IterGraph> graphs;
    IterGraph* capturing = nullptr;
    bool use_graphs = std::getenv("MGPBD_NO_GRAPH") == nullptr;

    void invalidate_graphs() {
        for (auto& g : graphs) {
            if (g.exec) cudaGraphExecDestroy(g.exec);
            for (auto& pr : g.ev) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
        }
        graphs.clear();
    }

    cudaEvent_t prof_event() {
        if (!capturing) return ev();
        cudaEvent_t e;
        MG_CK(cudaEventCreate(&e));
        return e;
    }

    void l0_pass(int mode, const T* xin, const T* b, T* y, const T* aux, double omega, double alpha = 0.0,
                 const T* xprev = nullptr, double x0_omega = 0.0, const std::function<void()>* mid = nullptr) {
        const Level& l0 = *L[0];
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        // inside stream capture a plain record is only a dependency: cudaEventRecordExternal makes it an event
        // record node whose timestamp the replay writes
        auto rec = [&](cudaEvent_t e) {
            if (capturing) MG_CK(cudaEventRecordWithFlags(e, st, cudaEventRecordExternal));
            else MG_CK(cudaEventRecord(e, st));
        };
        if (cfg.profile) { e0 = prof_event(); rec(e0); }
        if (mf_on()) mf_pass<T>(mode, mf, xin, b, y, aux, omega, parts1.p, parts2.p, st, alpha, xprev, x0_omega, mid);
        else csr_pass<T>(mode, l0.hot(), xin, b, y, aux, omega, parts1.p, parts2.p, st, alpha, xprev);
        if (cfg.profile) {
            e1 = prof_event();
            rec(e1);
            (capturing ? capturing->ev : prof_pairs).emplace_back(e0, e1);
            l0_launches++;
            l0_bytes_acc += pass_bytes(mode) - (x0_omega != 0.0 ? (double)sizeof(T) * (r1 - r0) : 0.0);  // x not read
        }
    }

    // alpha/xprev: the Chebyshev momentum of a smoother step (solve.cuh); 0 / nullptr otherwise
    void pass(int l, int mode, const T* xin, const T* b, T* y, const T* aux, double omega, double alpha = 0.0,
              const T* xprev = nullptr) {
        if (l == 0) {
            if (dist && mf_on() && halo_overlap && mf.vi1 > mf.vi0 && !xfers.empty()) {
                // partitioned matrix-free level 0: the halo exchange runs on a side stream while the interior
                // vertices (no halo incidence) are gathered; the boundary vertices and the rows wait for it
                if (!st_comm) {
                    MG_CK(cudaStreamCreateWithFlags(&st_comm, cudaStreamNonBlocking));
                    MG_CK(cudaEventCreateWithFlags(&ev_xa, cudaEventDisableTiming));
                    MG_CK(cudaEventCreateWithFlags(&ev_xb, cudaEventDisableTiming));
                }
                MG_CK(cudaEventRecord(ev_xa, st));
                MG_CK(cudaStreamWaitEvent(st_comm, ev_xa, 0));
                comm->exchange(const_cast<T*>(xin), sizeof(T), xfers, st_comm);
                MG_CK(cudaEventRecord(ev_xb, st_comm));
                const std::function<void()> mid = [&] { MG_CK(cudaStreamWaitEvent(st, ev_xb, 0)); };
                l0_pass(mode, xin, b, y, aux, omega, alpha, xprev, 0.0, &mid);
                return;
            }
            // partitioned level 0: bring the halo columns of x from the owning ranks first
            if (dist) comm->exchange(const_cast<T*>(xin), sizeof(T), xfers, st);
            l0_pass(mode, xin, b, y, aux, omega, alpha, xprev);
        }
        else csr_pass<T>(mode, L[l]->hot(), xin, b, y, aux, omega, parts1.p, parts2.p, st, alpha, xprev);
    }

    // Smoother coefficients of level a from lambda_max(D^-1 A) (lazily, at setup: PAPER.md:320).
    // Step k: x_{k+1} = x_k + alpha_k (x_k - x_{k-1}) + omega_k D^-1 (b - A x_k).
    //   omega-Jacobi: omega_k = 2/(s lambda + lambda_min_est), alpha_k = 0 (c9);
    //   Chebyshev on [lo, hi] = [cheb_lower hi, s lambda] (reading c20, Saad Alg. 12.1 with
    //   d_{k-1} = x_k - x_{k-1}): omega_0 = 1/theta, alpha_0 = 0, rho_0 = delta/theta,
    //   rho_k = 1/(2 theta/delta - rho_{k-1}), alpha_k = rho_k rho_{k-1}, omega_k = 2 rho_k/delta.
    void set_smoother(Level& a, double lam) {
        a.omega = 2.0 / (cfg.lambda_safety * lam + cfg.lambda_min_est);
        for (int k = 0; k < 8; ++k) { a.sm_omega[k] = a.omega; a.sm_alpha[k] = 0.0; }
        if (cfg.smoother == 1) {
            const double hi = cfg.lambda_safety * lam, lo = cfg.cheb_lower * hi;
            const double theta = 0.5 * (hi + lo), delta = 0.5 * (hi - lo), sigma = theta / delta;
            double rho = 1.0 / sigma;
            a.sm_omega[0] = 1.0 / theta;
            a.sm_alpha[0] = 0.0;
            for (int k = 1; k < 8; ++k) {
                const double rn = 1.0 / (2.0 * sigma - rho);
                a.sm_alpha[k] = rn * rho;
                a.sm_omega[k] = 2.0 * rn / delta;
                rho = rn;
            }
        }
    }

    void keep_power_iterate(Level& a) {
        a.pwv.resize(a.n);
        d2d(a.pwv.p, pw_v.p, a.n, st);
    }

    // Reading c26 (cfg.omega_refresh_iters > 0): at ite 0 of a frame without a setup,
    // lambda_max(D^-1 A_l) of every smoothed level is re-estimated on the CURRENT matrices with
    // omega_refresh_iters further power iterations started from the iterate the setup (or the previous
    // refresh) left, and the smoother coefficients and coarse-kernel tables follow.  The level matrices are
    // the fp64 ones the setup uses (A_0 from assemble_setup, the coarse levels by the fp64 Galerkin product
    // over the setup's aggregates / P), so the estimate matches the oracle's orc_hier_refresh_omega.
    void omega_refresh(double dt) {
        const int32_t iters = cfg.omega_refresh_iters;
        assemble_setup(dt);
        const bool mf0 = mf64_ok && mf_ready && h64.n;
        if (va_setup0) {
            at64.resize(m);
            va_at(m, alpha.p, last_dt, at64.p, st);
        }
        for (int l = 0; l + 1 < nL; ++l) {  // fp64 Galerkin values of levels 1..nL-1 (Eq. 6)
            Level& a = *L[l];
            Level& c = *L[l + 1];
            if (a.kk > 1)
                kgal_numeric<double>(a.plan, a.rowptr, a.col, a.val64.p, a.kk, a.kp.pptr.p, a.kp.pval64.p, a.kp.coff.p,
                                     a.agg.p, a.n_agg, a.erow.p, a.acol.p, a.xoff.p, c.rowptr, c.n, a.kW64.p, c.val64.p,
                                     c.dinv64.p, st);
            else if (l == 0 && va_setup0)
                va_numeric<double>(va, kc, h64.p, nullptr, a.P64.p, a.mptr.p, a.mlist.p, at64.p, a.n_agg, c.rowptr,
                                   c.val64.p, c.dinv64.p, st);
            else
                galerkin_numeric<double>(a.plan, a.rowptr, a.col, a.val64.p, a.P64.p, a.n_agg, c.rowptr, c.nnz,
                                         a.tval64.p, c.val64.p, c.dinv64.p, st);
        }
        for (int l = 0; l + 1 < nL; ++l) {
            Level& a = *L[l];
            if (!a.pwv.n) continue;
            double lam;
            if (l == 0 && mf0) {
                mf64.h = h64.p;
                mf64.dinv = a.dinv64.p;
                mf_refresh<double>(mf64, alpha.p, last_dt, a.dinv64.p, st);
                lam = power_method_op(
                    m, a.grid,
                    [&](const double* xv, double* yv, double* pp) {
                        mf_pass<double>(PASS_POWER, mf64, xv, nullptr, yv, nullptr, 0.0, pp, nullptr, st);
                        return mf64.grid;
                    },
                    iters, cfg.seed, l, a.pwv.p, pw_w.p, parts1.p, pw_ss.p, st, false);
            } else {
                lam = power_method(a.setup_csr(), iters, cfg.seed, l, a.pwv.p, pw_w.p, parts1.p, pw_ss.p, st, false);
            }
            set_smoother(a, lam);
        }
        plan_coarse();
        invalidate_graphs();  // the smoother coefficients are launch arguments of the captured iteration
        omega_refreshes++;
    }

    // The coarse-cycle kernels' tables (levels, smoother coefficients, resident / tail plans) from the current
    // hierarchy: at setup, and after a per-frame omega refresh (reading c26).
    // Reading c27: the first coarse level l >= 1 with at most `dense_cut` rows (and levels below it) becomes the
    // hot cycle's dense bottom z = M b, M rebuilt from the sub-cycle at every refresh (subcycle.cuh).
    void plan_subcycle() {
        sub_ok = false;
        lcut = -1;
        if (dense_cut <= 0 || kk != 1 || cfg.smoother == 2 || nL < 3) return;
        for (int l = 1; l + 1 < nL; ++l)
            if (L[l]->n <= dense_cut) { lcut = l; break; }
        if (lcut < 0 || nL - lcut > SUB_MAXL) { lcut = -1; return; }
        subc = SubCycle<T>();
        subc.K = nL - lcut;
        subc.nu = cfg.smoother_sweeps;
        subc.Ainv = Ainv.p;
        for (int l = lcut; l < nL; ++l) {
            Level& a = *L[l];
            SubLevel<T>& c = subc.L[l - lcut];
            c.n = a.n; c.nnz = (int32_t)a.nnz; c.rowptr = a.rowptr; c.col = a.col; c.val = a.val.p; c.dinv = a.dinv.p;
            for (int k = 0; k < 8; ++k) { c.om[k] = a.sm_omega[k]; c.al[k] = a.sm_alpha[k]; }
            if (l + 1 < nL) { c.agg = a.agg.p; c.P = a.P.p; c.mptr = a.mptr.p; c.mlist = a.mlist.p; c.n_next = a.n_agg; }
        }
        if (!subcycle_plan<T>(subc, 224u * 1024u)) { lcut = -1; return; }
        Mcut.resize((size_t)L[lcut]->n * L[lcut]->n);
        sub_ok = true;
    }
    // the hot cycle's bottom level (dense solve) and its matrix
    int lc() const { return sub_ok ? lcut : nL - 1; }
    const double* bottom_inv() const { return sub_ok ? Mcut.p : Ainv.p; }

    void plan_coarse() {
        plan_subcycle();
        plan_coarse_kernels();
        if (sub_ok && ccyc_ok && use_res && !res_ok) {  // the dense bottom's slices do not fit: plain bottom
            sub_ok = false;
            lcut = -1;
            plan_coarse_kernels();
        }
    }

    void plan_coarse_kernels() {
        ccyc_ok = false;
        if (use_coarse_kernel && cfg.smoother != 2 && kk == 1 && ccyc_from >= 1 && lc() >= ccyc_from + 1) {
            ccyc = CoarseCycle<T>();
            ccyc.K = lc() + 1 - ccyc_from;
            ccyc.nu = cfg.smoother_sweeps;
            ccyc.Ainv = bottom_inv();
            if (std::getenv("MGPBD_TRACE_COARSE")) {
                ctrace.resize(128);  // [0, 32): grid-wide kernel (down half), [32, 64): cluster tail, [64, 96): up half
                MG_CK(cudaMemsetAsync(ctrace.p, 0, 128 * sizeof(unsigned long long), st));
                ccyc.trace = ctrace.p;
            }
            for (int l = ccyc_from; l <= lc(); ++l) {
                Level& a = *L[l];
                CoarseLevel<T>& c = ccyc.L[l - ccyc_from];
                c.n = a.n; c.rowptr = a.rowptr; c.col = a.col; c.val = a.val.p; c.dinv = a.dinv.p; c.omega = a.omega;
                for (int k = 0; k < 8; ++k) { c.sm_omega[k] = a.sm_omega[k]; c.sm_alpha[k] = a.sm_alpha[k]; }
                if (l < lc()) { c.agg = a.agg.p; c.P = a.P.p; c.mptr = a.mptr.p; c.mlist = a.mlist.p; c.n_agg = a.n_agg; }
                c.t = a.vt.p; c.b = a.vb.p; c.z = a.vz.p; c.x = a.vx.p; c.y = a.vy.p;
            }
            ccyc_ok = true;
            res_ok = false;
            if (use_res) {
                int sms = 148;
                MG_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg.device));
                std::vector<ResLevel> lv;
                std::vector<ResCopy> cp;
                std::vector<int32_t> nc;
                std::vector<uint32_t> tx;
                uint32_t smem = 0;
                // 227 KB minus the static descriptor copy; MGPBD_RES_CAP (bytes, tests) lowers it to force the
                // global-kernel fallback
                const uint32_t cap = std::getenv("MGPBD_RES_CAP") ? (uint32_t)std::atol(std::getenv("MGPBD_RES_CAP"))
                                                                    : 220u * 1024u;
                ResPlan solo_plan;
                // solo tail: correct but issue-bound on one SM (~2.5 us per phase for a 548-row level, measured):
                // opt-in with MGPBD_SOLO=1
                const bool want_solo = std::getenv("MGPBD_SOLO") != nullptr;
                if (coarse_res_plan<T>(ccyc, sms, cap, lv, cp, nc, tx, smem, st, true, want_solo ? &solo_plan : nullptr) &&
                    coarse_res_blocks_per_sm<T>(smem) >= 1) {  // else the global coarse kernel
                    res_plan = ResPlan();
                    if (want_solo && solo_plan.solo_first <= ccyc.K - 2 && solo_plan.solo[0].n > 0) {
                        res_plan.solo_first = solo_plan.solo_first;
                        for (int q = 0; q < SOLO_MAXL; ++q) res_plan.solo[q] = solo_plan.solo[q];
                    }
                    res_lv.resize(lv.size()); h2d(res_lv.p, lv.data(), lv.size(), st);
                    res_cp.resize(cp.size()); h2d(res_cp.p, cp.data(), cp.size(), st);
                    res_nc.resize(nc.size()); h2d(res_nc.p, nc.data(), nc.size(), st);
                    res_tx.resize(tx.size()); h2d(res_tx.p, tx.data(), tx.size(), st);
                    res_plan.G = sms;
                    res_plan.smem = smem;
                    res_plan.lv = res_lv.p;
                    res_plan.copies = res_cp.p;
                    res_plan.ncopies = res_nc.p;
                    res_plan.txbytes = res_tx.p;
                    res_ok = true;
                }
            }
        }
        tail_ok = false;
        fused_ok = false;
        const bool solo_ok = res_ok && res_plan.solo[0].n > 0;
        // (the dense bottom of c27 leaves too little for a cluster tail to win: grid-only cycle)
        if (ccyc_ok && res_ok && use_tail && !solo_ok && !sub_ok) setup_tail();
        if (tracing)
            std::fprintf(stderr, "[mgpbd trace] levels %d coarse kernel %s from level %d, smem %u B, solo from %d, tail %s\n", nL,
                         !ccyc_ok ? "off" : res_ok ? "resident" : "global", ccyc_from, res_ok ? res_plan.smem : 0u,
                         solo_ok ? res_plan.solo_first : -1,
                         tail_ok ? (std::string(fused_ok ? "fused, " : "split, ") + "from cycle level " +
                                    std::to_string(fused_ok ? tail_f.first : tail.first) + " on " +
                                    std::to_string(fused_ok ? tail_f.CT : tail.CT) + " CTAs, " +
                                    std::to_string(fused_ok ? tail_f.smem : tail.smem) + " B" +
                                    (fused_ok ? ", grid " + std::to_string(res_f.G) : std::string())).c_str() : "off");
    }

    // ------------------------------------------------------------------ setup (Fig. setup-pipline)
    void setup() {
        Level& l0 = *L[0];
        L.resize(1);
        nL = 1;
        B0.resize(m);
        DBuf<double> B, Bn;
        const int maxl = std::min<int>(cfg.max_levels, MGPBD_MAX_LEVELS);
        pw_v.resize(m); pw_w.resize(m);
        bool va_built = false;
        trace(nullptr);
        for (int l = 0; l + 1 < maxl; ++l) {
            Level& a = *L[l];
            if (a.n < cfg.min_coarse) break;
            DBuf<uint8_t> strong;
            strong.resize(a.nnz);
            soc(a.n, a.rowptr, a.col, a.val64.p, cfg.theta, strong.p, st);
            trace("soc", l);
            a.agg.resize(a.n);
            int32_t na = aggregate(a.n, a.rowptr, a.col, a.val64.p, strong.p, cfg.seed, l, a.agg.p, st);
            trace("aggregate", l);
            if ((double)na > cfg.stall_ratio * (double)a.n) break;
            if (l == 0) {
                if (!colours_cached) {  // pattern fixed for the context lifetime: colour once
                    colours0.resize(a.n);
                    ncolours = colour(a.n, a.rowptr, a.col, cfg.seed, colours0.p, st);
                    colours_cached = true;
                    trace("colour", l);
                }
                const DBuf<int32_t>& col_ = colours0;
                B.resize((size_t)a.n * kk);
                GsOperator gop;
                const bool gs_mf = cfg.level0_operator == 1 && mf_ready && h64.n && !va_off;
                if (gs_mf) {  // the sweeps through H H^T + diag(at) (fp64 setup values)
                    at64.resize(m);
                    va_at(m, alpha.p, last_dt, at64.p, st);
                    gop.kc = kc; gop.nv = nv; gop.verts = verts.p; gop.h = h64.p; gop.vptr = vptr.p;
                    gop.vlist = vlist.p; gop.at = at64.p; gop.dinv = a.dinv64.p;
                }
                for (int c = 0; c < kk; ++c)  // k columns: hash index offset c n (reading c23)
                    gs_bootstrap(a.n, a.rowptr, a.col, a.val64.p, col_.p, ncolours, cfg.bootstrap_sweeps, cfg.seed,
                                 B.p + (size_t)c * a.n, st, gs_mf ? &gop : nullptr, (uint64_t)c * (uint64_t)a.n);
                B0.resize((size_t)m * kk);
                d2d(B0.p, B.p, (size_t)a.n * kk, st);
                trace("gs_bootstrap", l);
            }
            a.n_agg = na;
            if (cfg.smoother == 2) {  // multicolour GS order of this level (reading c22)
                DBuf<int32_t> cl, cnt_;
                const int32_t* cols = nullptr;
                if (l == 0) { cols = colours0.p; a.gs_ncol = ncolours; }
                else { cl.resize(a.n); a.gs_ncol = colour(a.n, a.rowptr, a.col, cfg.seed, cl.p, st); cols = cl.p; }
                group_by_key(cols, a.n, a.gs_ncol, a.gs_ptr, a.gs_list, cnt_, st, true);
                MG_CK(cudaStreamSynchronize(st));
            }
            DBuf<int32_t> cnt;
            group_by_key(a.agg.p, a.n, na, a.mptr, a.mlist, cnt, st, true);
            if (kk > 1) {  // k columns: per-aggregate QR injection (readings c24, c25)
                a.kk = kk;
                const int32_t nc = qr_prolongator(a.n, na, kk, a.agg.p, a.mptr.p, a.mlist.p, B.p, 1e-10, a.kp, Bn, st);
                trace("members+qr_prolongator", l);
                if ((double)nc > cfg.stall_ratio * (double)a.n) { a.kk = 1; break; }  // coarse DOFs decide (c7)
                galerkin_symbolic(a.n, a.rowptr, a.col, a.agg.p, a.mptr.p, a.mlist.p, na, a.plan, a.arow, a.acol, st);
                L.emplace_back(new Level());
                Level& c = *L[l + 1];
                Level& a2 = *L[l];
                kgal_expand(na, a2.arow.p, a2.acol.p, a2.kp.coff.p, c.rowptr_own, c.col_own, a2.xoff, a2.erow, st);
                c.n = nc;
                c.nnz = read_scalar(c.rowptr_own.p + nc, st);
                c.rowptr = c.rowptr_own.p; c.col = c.col_own.p;
                c.configure(st);
                c.val64.resize(c.nnz); c.dinv64.resize(c.n);
                a2.kW64.resize((size_t)std::max<int64_t>(a2.plan.T, 1) * kk);
                kgal_numeric<double>(a2.plan, a2.rowptr, a2.col, a2.val64.p, kk, a2.kp.pptr.p, a2.kp.pval64.p,
                                     a2.kp.coff.p, a2.agg.p, na, a2.erow.p, a2.acol.p, a2.xoff.p, c.rowptr, nc,
                                     a2.kW64.p, c.val64.p, c.dinv64.p, st);
                trace("k-galerkin", l);
                double lam;
                if (l == 0 && mf64_ok && mf_ready && h64.n) {
                    mf64.h = h64.p;
                    mf64.dinv = a2.dinv64.p;
                    mf_refresh<double>(mf64, alpha.p, last_dt, a2.dinv64.p, st);
                    lam = power_method_op(
                        m, a2.grid,
                        [&](const double* xv, double* yv, double* pp) {
                            mf_pass<double>(PASS_POWER, mf64, xv, nullptr, yv, nullptr, 0.0, pp, nullptr, st);
                            return mf64.grid;
                        },
                        cfg.power_iters, cfg.seed, l, pw_v.p, pw_w.p, parts1.p, pw_ss.p, st);
                } else {
                    lam = power_method(a2.setup_csr(), cfg.power_iters, cfg.seed, l, pw_v.p, pw_w.p, parts1.p, pw_ss.p, st);
                }
                keep_power_iterate(a2);
                set_smoother(a2, lam);
                trace("power", l);
                B.swap(Bn);
                nL = l + 2;
                pw_v.resize(std::max<size_t>(pw_v.n, (size_t)nc)); pw_w.resize(std::max<size_t>(pw_w.n, (size_t)nc));
                continue;
            }
            a.P64.resize(a.n);
            Bn.resize(na);
            prolongator(na, a.mptr.p, a.mlist.p, B.p, a.P64.p, Bn.p, st);
            trace("members+prolongator", l);
            L.emplace_back(new Level());
            Level& c = *L[l + 1];
            Level& a2 = *L[l];  // re-bind after emplace (unique_ptr: stable)
            // matrix-free level 0: P^T A_0 P from the fp64 gradients (vertex-aggregate form, vagal.cuh) — no
            // CSR Galerkin plan over the 1.4 GB level-0 pattern; the VA plan is the hot loop's as well
            const bool va_setup = l == 0 && cfg.level0_operator == 1 && mf_ready && h64.n && !va_off && kk == 1;
            if (va_setup) {
                GalerkinPlan& gp = a2.plan;  // not used: drop a CSR plan left by an earlier setup
                gp.gperm.free_all(); gp.tptr.free_all(); gp.tstart.free_all(); gp.trow.free_all();
                gp.tagg.free_all(); gp.lptr.free_all(); gp.llist.free_all(); gp.T = 0;
                va_coarse_pattern(nv, kc, vptr.p, vlist.p, a2.agg.p, na, c.rowptr_own, c.col_own, st);
                trace("va_pattern", l);
            } else {
                galerkin_symbolic(a2.n, a2.rowptr, a2.col, a2.agg.p, a2.mptr.p, a2.mlist.p, na, a2.plan, c.rowptr_own,
                                  c.col_own, st);
                trace("galerkin_symbolic", l);
            }
            c.n = na;
            c.nnz = read_scalar(c.rowptr_own.p + na, st);
            c.rowptr = c.rowptr_own.p; c.col = c.col_own.p;
            c.configure(st);
            c.val64.resize(c.nnz); c.dinv64.resize(c.n);
            if (va_setup) {
                va_symbolic(nv, kc, vptr.p, vlist.p, a2.agg.p, na, c.rowptr, c.col, c.nnz, va, st,
                            mf_ppos.n ? mf_ppos.p : nullptr, mf_npad);
                va_numeric<double>(va, kc, h64.p, nullptr, a2.P64.p, a2.mptr.p, a2.mlist.p, at64.p, na, c.rowptr, c.val64.p,
                                   c.dinv64.p, st);
                va_built = true;
                if (tracing)
                    std::fprintf(stderr, "[mgpbd trace] VA plan: %lld (vertex, aggregate) pairs, %lld products, %lld coarse entries\n",
                                 (long long)va.npairs, (long long)va.ncontrib, (long long)va.cnnz);
                trace("va_symbolic+numeric", l);
            } else {
                a2.tval64.resize(a2.plan.T);
                galerkin_numeric<double>(a2.plan, a2.rowptr, a2.col, a2.val64.p, a2.P64.p, na, c.rowptr, c.nnz,
                                         a2.tval64.p, c.val64.p, c.dinv64.p, st);
                trace("galerkin_numeric", l);
            }
            double lam;
            if (l == 0 && mf64_ok && mf_ready && h64.n) {
                // level 0 through the fp64 matrix-free operator (2 gathers instead of the 1.4 GB CSR)
                mf64.h = h64.p;
                mf64.dinv = a2.dinv64.p;
                mf_refresh<double>(mf64, alpha.p, last_dt, a2.dinv64.p, st);
                lam = power_method_op(
                    m, a2.grid,
                    [&](const double* xv, double* yv, double* pp) {
                        mf_pass<double>(PASS_POWER, mf64, xv, nullptr, yv, nullptr, 0.0, pp, nullptr, st);
                        return mf64.grid;
                    },
                    cfg.power_iters, cfg.seed, l, pw_v.p, pw_w.p, parts1.p, pw_ss.p, st);
            } else {
                lam = power_method(a2.setup_csr(), cfg.power_iters, cfg.seed, l, pw_v.p, pw_w.p, parts1.p, pw_ss.p, st);
            }
            keep_power_iterate(a2);
            set_smoother(a2, lam);
            trace("power", l);
            B.swap(Bn);
            nL = l + 2;
        }
        Level& cl = *L[nL - 1];
        if (cl.n > cfg.max_dense_coarse)
            throw Error(MGPBD_E_STALL, "coarsening stalled: coarsest level has " + std::to_string(cl.n) +
                                           " rows (> max_dense_coarse)");
        // hot buffers
        for (int l = 0; l < nL; ++l) {
            Level& a = *L[l];
            if (l > 0) { a.val.resize(a.nnz); a.dinv.resize(a.n); alloc_vectors(a); }
            if (l + 1 < nL && a.kk > 1) {
                a.kQs.resize((size_t)a.n * a.kk);
                convert<double, T>(a.kp.Qs64.p, a.kQs.p, (int64_t)a.n * a.kk, st);
                a.kpval.resize(a.kp.pcol.n);
                convert<double, T>(a.kp.pval64.p, a.kpval.p, (int64_t)a.kp.pcol.n, st);
                a.kW.resize((size_t)std::max<int64_t>(a.plan.T, 1) * a.kk);
                a.kones.resize(a.n);
                std::vector<T> ones((size_t)a.n, (T)1);
                h2d(a.kones.p, ones.data(), a.n, st);
            } else if (l + 1 < nL) {
                a.P.resize(a.n);
                convert<double, T>(a.P64.p, a.P.p, a.n, st);
                a.tval.resize(a.plan.T);
            }
        }
        if (dist && nL > 1 && !va_built) {  // level-0 Galerkin segments of the owned rows; the others stay zero
            Level& a = *L[0];
            tb0 = read_scalar(a.plan.tptr.p + r0, st);
            te0 = read_scalar(a.plan.tptr.p + r1, st);
            MG_CK(cudaMemsetAsync(a.tval.p, 0, sizeof(T) * (a.plan.T ? a.plan.T : 1), st));
        }
        va_ok = va_built && nL > 1;
        va_setup0 = va_built && nL > 1;
        if (!va_ok && cfg.level0_operator == 1 && nL > 1 && kk == 1) {
            va_symbolic(nv, kc, vptr.p, vlist.p, L[0]->agg.p, L[0]->n_agg, L[1]->rowptr, L[1]->col, L[1]->nnz, va, st,
                        mf_ppos.n ? mf_ppos.p : nullptr, mf_npad);
            va_ok = true;
            trace("va_symbolic");
        }
        Ainv.resize((size_t)cl.n * cl.n);
        inv_work.resize((size_t)cl.n * cl.n + 64 * (size_t)cl.n + 1024);
        plan_coarse();
        invalidate_graphs();  // buffers of the hierarchy changed
        have_hier = true;
        stale = false;
        (void)l0;
        MG_CK(cudaStreamSynchronize(st));
        trace("hot buffers");
    }

    // Cluster tail of the coarse cycle: plan it on 16 (else 8) CTAs; the top part of the cycle becomes a
    // truncated cycle (levels 0..first of ccyc, the last one only receiving b / providing z) run by the
    // resident kernel's down and up halves.
    bool setup_fused_tail() {
        const uint32_t cap = 220u * 1024u;
        for (int CT : {16, 8}) {
            if (!coarse_tail_plan<T>(ccyc, 1, CT, 110u * 1024u, tail_f, st)) continue;
            const int G = coarse_res_fused_grid<T>(CT, cap);
            if (G < CT) continue;
            CoarseCycle<T> top = ccyc;
            top.K = tail_f.first + 1;
            std::vector<ResLevel> lv;
            std::vector<ResCopy> cp;
            std::vector<int32_t> nc;
            std::vector<uint32_t> tx;
            uint32_t smem = 0;
            const uint32_t tcap = cap - ((tail_f.smem + 127u) & ~127u);
            if (!coarse_res_plan<T>(top, G, tcap, lv, cp, nc, tx, smem, st, /*with_coarsest=*/false)) continue;
            tail_base_f = (smem + 127u) & ~127u;
            if (coarse_res_fused_grid<T>(CT, tail_base_f + tail_f.smem) < G) continue;
            rf_lv.resize(lv.size()); h2d(rf_lv.p, lv.data(), lv.size(), st);
            rf_cp.resize(cp.size()); h2d(rf_cp.p, cp.data(), cp.size(), st);
            rf_nc.resize(nc.size()); h2d(rf_nc.p, nc.data(), nc.size(), st);
            rf_tx.resize(tx.size()); h2d(rf_tx.p, tx.data(), tx.size(), st);
            res_f.G = G;
            res_f.smem = smem;
            res_f.lv = rf_lv.p; res_f.copies = rf_cp.p; res_f.ncopies = rf_nc.p; res_f.txbytes = rf_tx.p;
            ccyc_f = top;
            targs_f = coarse_tail_args<T>(ccyc, tail_f);
            MG_CK(cudaStreamSynchronize(st));
            return true;
        }
        return false;
    }

    void setup_tail() {
        int sms = 148;
        MG_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg.device));
        const uint32_t cap = 220u * 1024u;
        fused_ok = use_fused && setup_fused_tail();
        if (fused_ok) { tail_ok = true; return; }
        for (int CT : {16, 8}) {
            if (coarse_tail_plan<T>(ccyc, 1, CT, cap, tail, st) && coarse_tail_launchable<T>(CT, tail.smem)) {
                tail_ok = true;
                break;
            }
        }
        if (!tail_ok) return;
        ccyc_top = ccyc;
        ccyc_top.K = tail.first + 1;
        std::vector<ResLevel> lv;
        std::vector<ResCopy> cp;
        std::vector<int32_t> nc;
        std::vector<uint32_t> tx;
        uint32_t smem = 0;
        if (!coarse_res_plan<T>(ccyc_top, sms, cap, lv, cp, nc, tx, smem, st, /*with_coarsest=*/false) ||
            coarse_res_blocks_per_sm<T>(smem) < 1) {
            tail_ok = false;
            return;
        }
        rt_lv.resize(lv.size()); h2d(rt_lv.p, lv.data(), lv.size(), st);
        rt_cp.resize(cp.size()); h2d(rt_cp.p, cp.data(), cp.size(), st);
        rt_nc.resize(nc.size()); h2d(rt_nc.p, nc.data(), nc.size(), st);
        rt_tx.resize(tx.size()); h2d(rt_tx.p, tx.data(), tx.size(), st);
        res_top.G = sms;
        res_top.smem = smem;
        res_top.lv = rt_lv.p;
        res_top.copies = rt_cp.p;
        res_top.ncopies = rt_nc.p;
        res_top.txbytes = rt_tx.p;
        MG_CK(cudaStreamSynchronize(st));
    }

    // MGPBD_TRACE=1: host wall time of the setup phases (stream synchronised at every mark).
    bool tracing = std::getenv("MGPBD_TRACE") != nullptr;
    std::chrono::steady_clock::time_point tr0;
    void trace(const char* what, int l = -1) {
        if (!tracing) return;
        MG_CK(cudaStreamSynchronize(st));
        auto now = std::chrono::steady_clock::now();
        if (what)
            std::fprintf(stderr, "[mgpbd trace] %-22s l=%2d %10.2f ms\n", what, l,
                         std::chrono::duration<double, std::milli>(now - tr0).count());
        tr0 = now;
    }

    // Galerkin values of all coarse levels from the current level-0 values + coarsest inverse.
    void refresh() {
        for (int l = 0; l + 1 < nL; ++l) {
            Level& a = *L[l];
            Level& c = *L[l + 1];
            if (a.kk > 1) {  // block Galerkin of the k > 1 hierarchy (nullspace.cuh) from the level's CSR values
                if (l == 0 && mf_on())  // the hot loop is matrix-free: assemble A_0's values for the product
                    assemble<T>(kind, m, verts.p, h.p, alpha.p, last_dt, rowptr0.p, col0.p, a.vl, a.val.p, a.dinv.p, st,
                                r0, r1);
                kgal_numeric<T>(a.plan, a.rowptr, a.col, a.val.p, a.kk, a.kp.pptr.p, a.kpval.p, a.kp.coff.p, a.agg.p,
                                a.n_agg, a.erow.p, a.acol.p, a.xoff.p, c.rowptr, c.n, a.kW.p, c.val.p, c.dinv.p, st);
                if (l == 0) mark_stage(1);
                continue;
            }
            if (l == 0 && va_ok && mf_on()) {  // from h directly (replicated on every rank, no collective)
                va_numeric<T>(va, kc, h.p, (mf.p0 == 0 && mf.p1 == mf.npad) ? (const T*)mf.hv : nullptr, a.P.p, a.mptr.p,
                              a.mlist.p, mf.at, a.n_agg, c.rowptr, c.val.p, c.dinv.p, st);
                mark_stage(1);
                continue;
            }
            if (l == 0 && dist) {  // this rank's fine rows only, then sum the partial coarse values
                galerkin_numeric<T>(a.plan, a.rowptr, a.col, a.val.p, a.P.p, a.n_agg, c.rowptr, c.nnz, a.tval.p,
                                    c.val.p, nullptr, st, tb0, te0);
                comm->allreduce(c.val.p, (size_t)c.nnz, st);
                diag_inv<T>(c.n, c.rowptr, c.val.p, c.dinv.p, st);
                mark_stage(1);
                continue;
            }
            galerkin_numeric<T>(a.plan, a.rowptr, a.col, a.val.p, a.P.p, a.n_agg, c.rowptr, c.nnz, a.tval.p, c.val.p,
                                c.dinv.p, st);
            if (l == 0) mark_stage(1);  // (stage stamps: level-0 product done)
        }
        mark_stage(2);
        coarse_invert<T>(L[nL - 1]->hot(), inv_work.p, Ainv.p, flags.p, st);
        if (sub_ok) subcycle_matrix<T>(subc, Mcut.p, st);  // reading c27
    }

    // ------------------------------------------------------------------ V-cycle
    // x_out = V(b) at level l, x = 0 start; at l = 0 with dot_r != nullptr the last post sweep also
    // produces the partials of r.z and r.r.
    void vcycle(int l, const T* b, T* x_out, const T* dot_r) {
        Level& a = *L[l];
        if (l == lc()) {  // coarsest: its inverse; or the dense bottom M of reading c27
            coarse_gemv<T>(a.n, bottom_inv(), b, x_out, st);
            return;
        }
        if (l == ccyc_from && ccyc_ok && b == a.vb.p && x_out == a.vz.p) {
            if (fused_ok) {  // one cooperative + cluster launch: grid down half, tail on cluster 0, grid up half
                coarse_vcycle_res<T>(ccyc_f, res_f, st, 3, tail_f.first, &targs_f, tail_base_f, tail_f.smem);
            } else if (tail_ok) {  // grid-wide down half, cluster tail, grid-wide up half
                coarse_vcycle_res<T>(ccyc_top, res_top, st, 1, tail.first);
                coarse_tail_run<T>(ccyc, tail, st);
                CoarseCycle<T> up = ccyc_top;
                if (up.trace) up.trace += 64;
                coarse_vcycle_res<T>(up, res_top, st, 2, tail.first);
            } else if (res_ok) {
                coarse_vcycle_res<T>(ccyc, res_plan, st);
            } else {
                coarse_vcycle<T>(ccyc, st);
            }
            return;
        }
        const int nu = cfg.smoother_sweeps;
        T* cur = a.vx.p;
        T* nxt = a.vy.p;
        const int32_t o = lo0(l), cn = cnt(l);  // rows this rank updates at this level
        if (cfg.smoother == 2) {  // multicolour GS: forward pre-sweeps, reversed post-sweeps (c22)
            const Csr<T> A = a.hot();
            MG_CK(cudaMemsetAsync(cur, 0, sizeof(T) * a.n, st));
            for (int sw = 0; sw < nu; ++sw) gs_sweep<T>(A, a.gs_ptr.p, a.gs_list.p, a.gs_ncol, false, b, cur, st);
            Level& c = *L[l + 1];
            if (a.kk > 1) {
                pass(l, PASS_RESID_P, cur, b, a.vt.p, a.kones.p, 0.0);
                krestrict<T>(c.n, a.kk, a.kp.dof_agg.p, a.kp.coff.p, a.mptr.p, a.mlist.p, a.kQs.p, a.vt.p, c.vb.p, st);
                vcycle(l + 1, c.vb.p, c.vz.p, nullptr);
                kprolong<T>(o, cn, a.kp.pptr.p, a.kp.pcol.p, a.kpval.p, c.vz.p, cur, st);
            } else {
                pass(l, PASS_RESID_P, cur, b, a.vt.p, a.P.p, 0.0);
                restrict_members<T>(a.n_agg, a.mptr.p, a.mlist.p, a.vt.p, c.vb.p, st);
                vcycle(l + 1, c.vb.p, c.vz.p, nullptr);
                prolong_add<T>(cn, a.agg.p + o, a.P.p + o, c.vz.p, cur + o, st);
            }
            for (int sw = 0; sw < nu; ++sw) gs_sweep<T>(A, a.gs_ptr.p, a.gs_list.p, a.gs_ncol, true, b, cur, st);
            d2d(x_out, cur, a.n, st);
            if (dot_r) {  // the partials of r.z and r.r the PCG finalisation expects
                dot_parts<T>(a.n, dot_r, x_out, parts1.p, l0_nparts(), st);
                dot_parts<T>(a.n, dot_r, dot_r, parts2.p, l0_nparts(), st);
            }
            return;
        }
        if (l == 0 && nu == 2 && fuse_jacobi0 && mf_on() && !dist && mf.tma && mf.vg_ts == 0) {
            // steps 0 and 1 in one matrix pass: x_1 = omega_0 D^-1 b is formed inside the gathers (no k_jacobi0
            // launch, no x_1 stream); same expressions, same result
            l0_pass(PASS_JACOBI, nullptr, b, nxt, nullptr, a.sm_omega[1], a.sm_alpha[1], nullptr, a.sm_omega[0]);
            std::swap(cur, nxt);
        } else {
            if (!(l == 0 && l0_x1_ready && b == r.p))  // (else formed by the previous x / r update)
                vec_jacobi0<T>(cn, a.dinv.p + o, b + o, a.sm_omega[0], cur + o, st);  // step 0 from x = 0
            if (l == 0) l0_x1_ready = false;
            for (int sw = 1; sw < nu; ++sw) {  // x_{sw+1} over x_{sw-1} (x_0 = 0: no xprev)
                pass(l, PASS_JACOBI, cur, b, nxt, nullptr, a.sm_omega[sw], a.sm_alpha[sw], sw == 1 ? nullptr : nxt);
                std::swap(cur, nxt);
            }
        }
        if (l == 0 && vc_trace) mark_stage(10);
        Level& c = *L[l + 1];
        if (a.kk > 1) {  // general P (k > 1): r = b - A x, b_c = P^T r, x += P e
            pass(l, PASS_RESID_P, cur, b, a.vt.p, a.kones.p, 0.0);
            if (l == 0 && vc_trace) mark_stage(11);
            krestrict<T>(c.n, a.kk, a.kp.dof_agg.p, a.kp.coff.p, a.mptr.p, a.mlist.p, a.kQs.p, a.vt.p, c.vb.p, st);
            if (l == 0 && vc_trace) mark_stage(12);
            vcycle(l + 1, c.vb.p, c.vz.p, nullptr);
            if (l == 0 && vc_trace) mark_stage(13);
            kprolong<T>(o, cn, a.kp.pptr.p, a.kp.pcol.p, a.kpval.p, c.vz.p, cur, st);
            if (l == 0 && vc_trace) mark_stage(14);
        } else {
            pass(l, PASS_RESID_P, cur, b, a.vt.p, a.P.p, 0.0);
            if (l == 0 && vc_trace) mark_stage(11);
            restrict_members<T>(a.n_agg, a.mptr.p, a.mlist.p, a.vt.p, c.vb.p, st);
            if (l == 0 && dist) comm->allreduce(c.vb.p, (size_t)c.n, st);  // partial sums of split aggregates
            if (l == 0 && vc_trace) mark_stage(12);
            vcycle(l + 1, c.vb.p, c.vz.p, nullptr);
            if (l == 0 && vc_trace) mark_stage(13);
            prolong_add<T>(cn, a.agg.p + o, a.P.p + o, c.vz.p, cur + o, st);
            if (l == 0 && vc_trace) mark_stage(14);
        }
        for (int sw = 0; sw < nu; ++sw) {
            const bool last = sw == nu - 1;
            T* other = cur == a.vx.p ? a.vy.p : a.vx.p;  // holds x_{sw-1} for sw >= 1
            T* dst = last ? x_out : other;
            const T* xprev = sw == 0 ? nullptr : other;
            if (last && dot_r) pass(l, PASS_JACOBI_DOT, cur, b, dst, dot_r, a.sm_omega[sw], a.sm_alpha[sw], xprev);
            else pass(l, PASS_JACOBI, cur, b, dst, nullptr, a.sm_omega[sw], a.sm_alpha[sw], xprev);
            if (l == 0 && vc_trace) mark_stage(15 + std::min(sw, 1));
            cur = dst;
        }
    }

    // ------------------------------------------------------------------ MGPCG
    void pcg(int32_t iters, int ite) {
        Level& l0 = *L[0];
        MG_CK(cudaMemsetAsync(xs.p, 0, sizeof(T) * m, st));
        pcg_begin(scal.p, cfg.pcg_tol, st);  // convergence exit state (pcg_tol; off by default)
        d2d(r.p, b0.p, m, st);
        MG_CK(cudaMemsetAsync(p.p, 0, sizeof(T) * m, st));
        T* z = l0.vz.p;
        const int32_t o = r0, cn = r1 - r0;
        if (dist && nL == 1) throw Error(MGPBD_E_ARG, "a partitioned solve needs at least two levels");
        for (int k = 0; k < iters; ++k) {
            const int tag = k;  // + flags[7] (outer iteration) * 4096, added on the device
            if (nL == 1) {
                vcycle(0, r.p, z, nullptr);
                dot_parts<T>(m, r.p, z, parts1.p, l0.grid, st);
                dot_parts<T>(m, r.p, r.p, parts2.p, l0.grid, st);
            } else {
                if (k == 0) mark_stage(6);
                vc_trace = k == 0 && trace_stages;
                timed(PH_VC, [&] { vcycle(0, r.p, z, r.p); });
                vc_trace = false;
                if (k == 0) mark_stage(7);
            }
            const int np = nL == 1 ? l0.grid : l0_nparts();
            if (dist) {  // rank-local sums -> allreduce -> checks on the global values
                finalize_sum(parts1.p, np, dsc.p, st);
                finalize_sum(parts2.p, np, dsc.p + 1, st);
                comm->allreduce(dsc.p, 2, st);
                pcg_commit_rz(dsc.p, scal.p, k, flags.p, tag, st);
                pcg_update_p<T>(cn, z + o, p.p + o, scal.p, k, st);
            } else {
                pcg_update_p_fin<T>(cn, z + o, p.p + o, scal.p, k, parts1.p, parts2.p, np, flags.p, tag, st, fin_ready());
            }
            if (k == 0) mark_stage(8);
            pass(0, PASS_SPMV_DOT, p.p, nullptr, q.p, nullptr, 0.0);
            if (k == 0) mark_stage(9);
            if (dist) {
                finalize_sum(parts1.p, l0_nparts(), dsc.p + 2, st);
                comm->allreduce(dsc.p + 2, 1, st);
                pcg_commit_pq(dsc.p + 2, scal.p, k, flags.p, tag, st);
                pcg_update_xr<T>(cn, p.p + o, q.p + o, xs.p + o, r.p + o, scal.p, k, st);
            } else {
                // the next iteration's V-cycle starts with x1 = omega_0 D^-1 r: formed here from the new r
                const bool x1 = k + 1 < iters && x1_fusable();
                pcg_update_xr_fin<T>(cn, p.p + o, q.p + o, xs.p + o, r.p + o, scal.p, k, parts1.p, l0_nparts(),
                                     flags.p, tag, st, l0.dinv.p + o, l0.sm_omega[0], x1 ? l0.vx.p + o : nullptr,
                                     fin_ready());
                l0_x1_ready = x1;
            }
            if (k == 0) mark_stage(17);
        }
    }

    void assemble_hot(double dt) {
        Level& l0 = *L[0];
        // one rank, matrix-free: the evaluation also writes hv / at / D^-1 (no k_mf_refresh pass over h)
        const bool fused = cfg.level0_operator == 1 && !dist && eval_hv && mf.p0 == 0 && mf.p1 == mf_npad &&
                           mf_inv.n == (size_t)m * kc && npad_fits();
        EvalHv<T> e;
        if (fused) { e.inv = mf_inv.p; e.hv = mf_hv.p; e.npad = mf_npad; e.at = mf_at.p; e.dinv = l0.dinv.p; }
        eval_constraints<T>(kind, m, verts.p, x.p, rest.p, sqrtw.p, alpha.p, dt, lambda.p, h.p, b0.p, st,
                            fused ? &e : nullptr);
        // (all constraints are evaluated on every rank: h of the halo constraints is needed locally)
        last_dt = dt;
        if (cfg.level0_operator == 1) {
            // matrix-free level 0: no assembled matrix in the hot loop (diagonal and A_1 from h)
            if (!fused) mf_refresh<T>(mf, alpha.p, dt, l0.dinv.p, st);
            mf_ready = true;
        } else {
            assemble<T>(kind, m, verts.p, h.p, alpha.p, dt, rowptr0.p, col0.p, l0.vl, l0.val.p, l0.dinv.p, st, r0, r1);
        }
    }

    void assemble_setup(double dt) {
        Level& l0 = *L[0];
        l0.val64.resize(nnz0);
        l0.dinv64.resize(m);
        if (std::is_same<T, double>::value && !dist && cfg.level0_operator == 0) {
            d2d(l0.val64.p, (const double*)l0.val.p, nnz0, st);
            d2d(l0.dinv64.p, (const double*)l0.dinv.p, m, st);
        } else {
            h64.resize((size_t)m * kc * 3); b64.resize(m);
            eval_constraints<double>(kind, m, verts.p, x.p, rest.p, sqrtw.p, alpha.p, dt, lambda.p, h64.p, b64.p, st);
            assemble<double>(kind, m, verts.p, h64.p, alpha.p, dt, rowptr0.p, col0.p, l0.vl, l0.val64.p, l0.dinv64.p, st);
        }
    }

    // stage timestamps of one outer iteration (MGPBD_TRACE_STAGES=1; printed at frame end)
    bool trace_stages = std::getenv("MGPBD_TRACE_STAGES") != nullptr;
    DBuf<unsigned long long> stamps;
    void mark_stage(int idx) {
        if (!trace_stages) return;
        if (stamps.n < 32) stamps.resize(32);
        stamp(stamps.p, idx, st);
    }

    void iter_body(int ite) {
        mark_stage(0);
        timed(PH_GAL, [&] { refresh(); });                                                           // Eq. 6
        mark_stage(3);
        timed(PH_PCG, [&] { pcg(cfg.pcg_iters, ite); });                                             // l.8
        mark_stage(4);
        timed(PH_UPD, [&] {
            if (dist) comm->allgather_blocks(xs.p, sizeof(T), part_bounds, st);  // dlambda of every row, every rank
            if (mf_on() && !dist && mf.p0 == 0 && mf.p1 == mf.npad)  // hv covers every incidence
                mf_update<T>(mf, xs.p, sqrtw.p, omega_dev.p, x.p, st);                       // l.9, l.11
            else
                update_positions<T>(nv, kc, vptr.p, vlist.p, h.p, sqrtw.p, xs.p, omega_dev.p, x.p, st);
            lambda_add<T>(m, lambda.p, xs.p, st);                                                    // l.10
        });
        mark_stage(5);
    }

    // 1: eager launches with CUDA events around every level-0 pass and phase; 2: the same pass events captured
    // as nodes of the per-iteration graph (the replayed frame as the bench times it; each replay overwrites
    // the events, so the last replay's pass durations stand for every outer iteration of the frame)
    bool graph_profile = false;
    void set_profiling(int on) override {
        const bool gp = on == 2;
        if (gp != graph_profile || (on != 0) != (cfg.profile != 0)) invalidate_graphs();
        graph_profile = gp;
        cfg.profile = on ? 1 : 0;
    }

    // One graph serves every outer iteration (the iteration index reaches the kernels through flags[7]),
    // so after a setup only the second outer iteration pays the capture + instantiation.
    void run_iter(int ite) {
        set_outer_index(flags.p, std::min(ite, 500000), st);  // error tags ite*4096 + k stay within int32
        if (!use_graphs || (cfg.profile && !graph_profile)) { iter_body(ite); return; }  // eager event timing
        if (graphs.empty()) graphs.resize(1);
        IterGraph& g = graphs[0];
        if (!g.seen) {  // first use after a (re)build: eager
            g.seen = true;
            iter_body(ite);
            return;
        }
        if (!g.exec) {
            const int64_t kl = g_kernel_launches, l0l = l0_launches;
            const double l0b = l0_bytes_acc;
            capturing = &g;
            MG_CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            iter_body(ite);
            cudaGraph_t graph;
            const cudaError_t ec = cudaStreamEndCapture(st, &graph);
            capturing = nullptr;
            MG_CK(ec);
            MG_CK(cudaGraphInstantiate(&g.exec, graph, 0));
            MG_CK(cudaGraphDestroy(graph));
            g.launches = g_kernel_launches - kl;
            g.l0_launches = l0_launches - l0l;
            g.l0_bytes = l0_bytes_acc - l0b;
            g_kernel_launches = kl; l0_launches = l0l; l0_bytes_acc = l0b;  // counted at replay
        }
        MG_CK(cudaGraphLaunch(g.exec, st));
        g_kernel_launches += g.launches;
        if (cfg.profile) {
            l0_launches += g.l0_launches;
            l0_bytes_acc += g.l0_bytes;
            for (auto& pr : g.ev) prof_pairs.push_back(pr);
        }
    }

    // ------------------------------------------------------------------ Algorithm 1
    void step(double dt, int32_t n_iters) override {
        ev_used = 0;
        l0_launches = 0;
        l0_bytes_acc = 0;
        setup_ran = 0;
        prof_pairs.clear();
        for (auto& v_ : ph_pairs) v_.clear();
        g_kernel_launches = 0;
        cudaEvent_t f0 = ev(), f1, s0 = nullptr, s1 = nullptr;
        MG_CK(cudaEventRecord(f0, st));
        MG_CK(cudaMemsetAsync(flags.p, 0, 8 * sizeof(int), st));
        predict(nv, x.p, v.p, x_old.p, w.p, dt, cfg.gravity[0], cfg.gravity[1], cfg.gravity[2], st);  // l.1
        omega_dev.resize(1);
        h2d(omega_dev.p, &cfg.omega_relax, 1, st);  // user omega; halved below if backtracking
        MG_CK(cudaMemsetAsync(lambda.p, 0, sizeof(double) * m, st));                                // l.2
        int32_t iters_run = 0;
        for (int ite = 0; ite < n_iters; ++ite) {                                                    // l.3
            timed(PH_ASM, [&] { assemble_hot(dt); });                                                // l.4-6
            dot_parts<T>(m, b0.p, b0.p, parts2.p, L[0]->grid, st);
            finalize_sum(parts2.p, L[0]->grid, bn.p + ite, st);
            if (cfg.backtrack) backtrack_omega(bn.p, ite, omega_dev.p, cfg.omega_min, st);
            if (ite == 0 && (stale || !have_hier || frame % cfg.setup_interval == 0)) {            // l.7
                s0 = ev();
                MG_CK(cudaEventRecord(s0, st));
                assemble_setup(dt);
                setup();
                s1 = ev();
                MG_CK(cudaEventRecord(s1, st));
                setup_ran = 1;
            } else if (ite == 0 && cfg.omega_refresh_iters > 0 && have_hier && nL > 1) {  // reading c26
                omega_refresh(dt);
            }
            if (cfg.level0_operator == 1 && nL < 2)  // single level: A_0 is the coarsest, inverted densely
                assemble<T>(kind, m, verts.p, h.p, alpha.p, dt, rowptr0.p, col0.p, L[0]->vl, L[0]->val.p,
                            L[0]->dinv.p, st, r0, r1);
            run_iter(ite);  // Eq. 6 refresh, l.8 MGPCG, l.9-11 update
            iters_run = ite + 1;
            if (cfg.residual_tol > 0.0 || cfg.residual_abs > 0.0) {
                // l.12: ||b|| < eps, eps = residual_tol ||b_0|| (reading c21) or residual_abs
                double b2[2];
                d2h(b2, bn.p, 1, st);
                d2h(b2 + 1, bn.p + ite, 1, st);
                MG_CK(cudaStreamSynchronize(st));
                if (cfg.residual_tol > 0.0 && b2[1] < cfg.residual_tol * cfg.residual_tol * b2[0]) break;
                if (cfg.residual_abs > 0.0 && b2[1] < cfg.residual_abs * cfg.residual_abs) break;
            }
            if (cfg.time_budget_ms > 0.0) {  // l.12 timeBudgetExhausted: device time since the frame started
                cudaEvent_t ei = ev();
                MG_CK(cudaEventRecord(ei, st));
                MG_CK(cudaEventSynchronize(ei));
                float el = 0.0f;
                MG_CK(cudaEventElapsedTime(&el, f0, ei));
                if ((double)el > cfg.time_budget_ms) break;
            }
        }
        velocity(nv, x.p, x_old.p, v.p, dt, st);                                                     // l.17
        f1 = ev();
        MG_CK(cudaEventRecord(f1, st));
        MG_CK(cudaStreamSynchronize(st));
        launches_last = g_kernel_launches;
        if (trace_stages && stamps.n) {  // stage times of the last outer iteration
            unsigned long long tt[18];
            d2h(tt, stamps.p, 18, st);
            MG_CK(cudaStreamSynchronize(st));
            auto us = [&](int a, int b) { return (double)(tt[b] - tt[a]) * 1e-3; };
            std::fprintf(stderr,
                         "[mgpbd stages] refresh: VA %.1f levels %.1f coarsest-inverse %.1f | pcg %.1f (first "
                         "iteration: V-cycle %.1f, p-update %.1f, SpMV %.1f, x/r-update %.1f) | update %.1f us\n",
                         us(0, 1), us(1, 2), us(2, 3), us(3, 4), us(6, 7), us(7, 8), us(8, 9), us(9, 17), us(4, 5));
            if (tt[10] && tt[16])
                std::fprintf(stderr,
                             "[mgpbd stages] level-0 V-cycle: pre-smoothing %.1f, residual %.1f, restriction %.1f, coarse "
                             "levels %.1f, prolongation %.1f, post step 1 %.1f, post step 2 %.1f us\n",
                             us(6, 10), us(10, 11), us(11, 12), us(12, 13), us(13, 14), us(14, 15), us(15, 16));
        }
        if (ccyc.trace) {  // phase times of the last coarse V-cycle (MGPBD_TRACE_COARSE)
            unsigned long long tt[128];
            d2h(tt, ctrace.p, 128, st);
            MG_CK(cudaStreamSynchronize(st));
            const char* names[3] = {"grid", "tail", "up"};
            unsigned long long prev_end = 0;
            for (int part = 0; part < 3; ++part) {
                const unsigned long long* p = tt + 32 * part;
                if (!p[0]) continue;
                int nmark = 1;
                while (nmark < 32 && p[nmark] >= p[nmark - 1] && p[nmark]) ++nmark;
                const unsigned long long entry = tt[96 + part];
                std::fprintf(stderr, "[mgpbd coarse] K=%d %s (gap %.2f us, staging %.2f us, %.2f us total) phases (us):",
                             ccyc.K, names[part], prev_end ? (double)(p[0] - prev_end) * 1e-3 : 0.0,
                             entry && entry <= p[0] ? (double)(p[0] - entry) * 1e-3 : 0.0, (double)(p[nmark - 1] - p[0]) * 1e-3);
                for (int k = 1; k < nmark; ++k) std::fprintf(stderr, " %.2f", (p[k] - p[k - 1]) * 1e-3);
                std::fprintf(stderr, "\n");
                prev_end = p[nmark - 1];
            }
        }
        frame++;
        n_b = iters_run;
        d2h(&omega_last, omega_dev.p, 1, st);
        float ms = 0;
        MG_CK(cudaEventElapsedTime(&ms, f0, f1));
        ms_frame = ms;
        ms_setup = 0;
        if (s0) { MG_CK(cudaEventElapsedTime(&ms, s0, s1)); ms_setup = ms; }
        if (cfg.profile) {
            double tot = 0;
            for (auto& pr : prof_pairs) {
                MG_CK(cudaEventElapsedTime(&ms, pr.first, pr.second));
                tot += ms;
            }
            l0_ms = tot;
            l0_bytes = l0_bytes_acc;
            for (int ph = 0; ph < PH_N; ++ph) {
                double t = 0;
                for (auto& pr : ph_pairs[ph]) {
                    MG_CK(cudaEventElapsedTime(&ms, pr.first, pr.second));
                    t += ms;
                }
                ph_ms[ph] = t;
            }
        } else {
            for (double& t : ph_ms) t = 0;
        }
        int hf[6];
        d2h(hf, flags.p, 6, st);
        MG_CK(cudaStreamSynchronize(st));
        // <z,r> <= 0: the lazily-set omega is no longer below 2/lambda_max -> re-run the setup at ite 0
        // of the next frame (reading c13; cfg.resetup_on_indef); counted, not an error.
        indef_events = hf[4];
        if (indef_events && cfg.resetup_on_indef) stale = true;
        if (hf[1]) throw Error(MGPBD_E_NONFINITE, "non-finite PCG scalar at (frame " + std::to_string(frame - 1) +
                                                      ", ite " + std::to_string(hf[3] / 4096) + ", pcg " +
                                                      std::to_string(hf[3] % 4096) + ")");
        if (hf[5]) throw Error(MGPBD_E_INDEFINITE, "non-SPD coarsest matrix in frame " + std::to_string(frame - 1));
    }

    void set_state(const double* pos, const double* vel) override {
        if (pos) h2d(x.p, pos, 3 * (size_t)nv, st);
        if (vel) h2d(v.p, vel, 3 * (size_t)nv, st);
        MG_CK(cudaStreamSynchronize(st));
    }
    void get_positions(double* out) override { d2h(out, x.p, 3 * (size_t)nv, st); MG_CK(cudaStreamSynchronize(st)); }
    void get_velocities(double* out) override { d2h(out, v.p, 3 * (size_t)nv, st); MG_CK(cudaStreamSynchronize(st)); }
    void get_lambda(double* out) override { d2h(out, lambda.p, m, st); MG_CK(cudaStreamSynchronize(st)); }

    void get_stats(mgpbd_stats* s) override {
        std::memset(s, 0, sizeof(*s));
        s->n_levels = have_hier ? nL : 0;
        double tot = 0;
        for (int l = 0; l < s->n_levels; ++l) {
            s->n[l] = L[l]->n; s->nnz[l] = L[l]->nnz; tot += (double)L[l]->nnz;
            s->omega[l] = L[l]->omega;
        }
        s->op_complexity = s->n_levels ? tot / (double)nnz0 : 0.0;
        s->n_colours = ncolours;
        s->setup_ran = setup_ran;
        s->n_b = n_b;
        const int nb = std::min(n_b, (int)MGPBD_MAX_ITERS);
        s->n_b = nb;
        s->iters_run = n_b;
        if (nb) d2h(s->b_norm, bn.p, nb, st);
        if (n_b) d2h(&s->b_last, bn.p + n_b - 1, 1, st);
        MG_CK(cudaStreamSynchronize(st));
        for (int i = 0; i < nb; ++i) s->b_norm[i] = std::sqrt(s->b_norm[i]);
        s->b_last = std::sqrt(s->b_last);
        s->frame = frame;
        s->l0_pass_ms = l0_ms;
        s->l0_pass_launches = cfg.profile ? l0_launches : 0;
        s->l0_pass_bytes = l0_bytes;
        s->ms_setup = ms_setup;
        s->ms_frame = ms_frame;
        s->kernel_launches = launches_last;
        s->indefinite_events = indef_events;
        s->rank = dist ? comm->rank() : 0;
        s->world = dist ? comm->world() : 1;
        s->row_begin = r0;
        s->row_end = r1;
        s->halo_rows = halo_elems;
        s->omega_relax = omega_last;
        s->ms_assemble = ph_ms[PH_ASM];
        s->ms_galerkin = ph_ms[PH_GAL];
        s->ms_vcycle = ph_ms[PH_VC];
        s->ms_pcg_other = ph_ms[PH_PCG] - ph_ms[PH_VC];
        s->ms_update = ph_ms[PH_UPD];
    }

    void check_level(int l) {
        if (l == 0) return;  // the level-0 pattern exists from mgpbd_create on
        if (!have_hier || l < 0 || l >= nL) throw Error(MGPBD_E_ARG, "level out of range (or no hierarchy yet)");
    }
    void level_sizes(int l, int64_t* n, int64_t* nnz) override {
        check_level(l);
        *n = L[l]->n; *nnz = L[l]->nnz;
    }

    void get_level(int l, int64_t* rp, int32_t* cl, double* vals) override {
        check_level(l);
        Level& a = *L[l];
        if (l == 0 && vals && cfg.level0_operator == 1 && last_dt > 0)  // not assembled in the hot loop
            assemble<T>(kind, m, verts.p, h.p, alpha.p, last_dt, rowptr0.p, col0.p, a.vl, a.val.p, a.dinv.p, st);
        if (rp) d2h(rp, a.rowptr, (size_t)a.n + 1, st);
        if (cl) d2h(cl, a.col, a.nnz, st);
        if (vals) {
            std::vector<T> tmp(a.nnz);
            d2h(tmp.data(), a.val.p, a.nnz, st);
            MG_CK(cudaStreamSynchronize(st));
            for (int64_t k = 0; k < a.nnz; ++k) vals[k] = (double)tmp[k];
        }
        MG_CK(cudaStreamSynchronize(st));
    }
    void get_prolongator_csr(int l, int64_t* nnz, int64_t* rp, int32_t* cl, double* vals) override {
        check_level(l);
        if (!have_hier || l >= nL - 1) throw Error(MGPBD_E_ARG, "coarsest level has no prolongator");
        const Level& a = *L[l];
        if (a.kk > 1) {
            *nnz = (int64_t)a.kp.pcol.n;
            if (rp) d2h(rp, a.kp.pptr.p, (size_t)a.n + 1, st);
            if (cl) d2h(cl, a.kp.pcol.p, a.kp.pcol.n, st);
            if (vals) d2h(vals, a.kp.pval64.p, a.kp.pcol.n, st);
        } else {
            *nnz = a.n;
            if (cl) d2h(cl, a.agg.p, a.n, st);
            if (vals) d2h(vals, a.P64.p, a.n, st);
            if (rp)
                for (int64_t i = 0; i <= a.n; ++i) rp[i] = i;
        }
        MG_CK(cudaStreamSynchronize(st));
    }
    void get_prolongator(int l, double* pv) override {
        check_level(l);
        if (!have_hier || l >= nL - 1) throw Error(MGPBD_E_ARG, "coarsest level has no prolongator");
        if (L[l]->kk > 1) throw Error(MGPBD_E_ARG, "k_nullspace > 1: use mgpbd_get_prolongator_csr");
        d2h(pv, L[l]->P64.p, L[l]->n, st);
        MG_CK(cudaStreamSynchronize(st));
    }
    void get_aggregates(int l, int32_t* ag) override {
        check_level(l);
        if (!have_hier || l >= nL - 1) throw Error(MGPBD_E_ARG, "coarsest level has no aggregates");
        d2h(ag, L[l]->agg.p, L[l]->n, st);
        MG_CK(cudaStreamSynchronize(st));
    }
    void get_near_kernel(double* bout) override {
        if (!have_hier || nL < 2) throw Error(MGPBD_E_ARG, "no bootstrapped near kernel (single-level hierarchy)");
        d2h(bout, B0.p, (size_t)m * kk, st);
        MG_CK(cudaStreamSynchronize(st));
    }
    void debug_setup_from(const double* vals) override {
        Level& l0 = *L[0];
        mf_ready = false;  // external A_0 values: h does not describe them, use the CSR passes
        l0.val64.resize(nnz0); l0.dinv64.resize(m);
        h2d(l0.val64.p, vals, nnz0, st);
        diag_inv<double>(m, rowptr0.p, l0.val64.p, l0.dinv64.p, st);
        convert<double, T>(l0.val64.p, l0.val.p, nnz0, st);
        diag_inv<T>(m, rowptr0.p, l0.val.p, l0.dinv.p, st);
        setup();
        refresh();
        MG_CK(cudaStreamSynchronize(st));
    }
    void debug_vcycle(const double* b, double* xo) override {
        if (!have_hier) throw Error(MGPBD_E_ARG, "no hierarchy");
        DBuf<double> tmp;
        tmp.resize(m);
        h2d(tmp.p, b, m, st);
        convert<double, T>(tmp.p, r.p, m, st);
        vcycle(0, r.p, L[0]->vz.p, nullptr);
        convert<T, double>(L[0]->vz.p, tmp.p, m, st);
        d2h(xo, tmp.p, m, st);
        MG_CK(cudaStreamSynchronize(st));
    }
    // `reps` level-0 SpMV+dot passes (the hot operator on the current state) captured into one CUDA
    // graph and timed with events around its launch (after one warm-up replay): the pass rate without
    // launch gaps.  Returns the device time of the replay and the passes' algorithmic bytes.
    void pass_burst(int32_t reps, double* ms, double* bytes) override {
        if (!have_hier || (cfg.level0_operator == 1 && !mf_ready)) throw Error(MGPBD_E_ARG, "no current state");
        if (dist) throw Error(MGPBD_E_ARG, "pass_burst: one rank only");
        cudaGraph_t graph;
        cudaGraphExec_t exec;
        const bool prof = cfg.profile;
        cfg.profile = 0;
        MG_CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        for (int k = 0; k < reps; ++k) l0_pass(PASS_SPMV_DOT, p.p, nullptr, q.p, nullptr, 0.0);
        const cudaError_t ec = cudaStreamEndCapture(st, &graph);
        cfg.profile = prof;
        MG_CK(ec);
        MG_CK(cudaGraphInstantiate(&exec, graph, 0));
        MG_CK(cudaGraphDestroy(graph));
        cudaEvent_t e0, e1;
        MG_CK(cudaEventCreate(&e0));
        MG_CK(cudaEventCreate(&e1));
        MG_CK(cudaGraphLaunch(exec, st));  // warm-up
        MG_CK(cudaEventRecord(e0, st));
        MG_CK(cudaGraphLaunch(exec, st));
        MG_CK(cudaEventRecord(e1, st));
        MG_CK(cudaEventSynchronize(e1));
        float t = 0;
        MG_CK(cudaEventElapsedTime(&t, e0, e1));
        *ms = t;
        *bytes = pass_bytes(PASS_SPMV_DOT) * reps;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaGraphExecDestroy(exec);
    }

    void debug_prepare(double dt) override {
        MG_CK(cudaMemsetAsync(flags.p, 0, 8 * sizeof(int), st));
        predict(nv, x.p, v.p, x_old.p, w.p, dt, cfg.gravity[0], cfg.gravity[1], cfg.gravity[2], st);  // l.1
        omega_dev.resize(1);
        h2d(omega_dev.p, &cfg.omega_relax, 1, st);
        MG_CK(cudaMemsetAsync(lambda.p, 0, sizeof(double) * m, st));                                // l.2
        assemble_hot(dt);                                                                            // l.4-6
        if (stale || !have_hier || frame % cfg.setup_interval == 0) {                               // l.7
            assemble_setup(dt);
            setup();
        } else if (cfg.omega_refresh_iters > 0 && have_hier && nL > 1) {
            omega_refresh(dt);  // reading c26
        }
        if (cfg.level0_operator == 1 && nL < 2)
            assemble<T>(kind, m, verts.p, h.p, alpha.p, dt, rowptr0.p, col0.p, L[0]->vl, L[0]->val.p,
                        L[0]->dinv.p, st, r0, r1);
        refresh();                                                                                   // Eq. 6
        MG_CK(cudaStreamSynchronize(st));
    }

    void debug_pcg(const double* b, int32_t iters, double* xo) override {
        if (!have_hier) throw Error(MGPBD_E_ARG, "no hierarchy");
        DBuf<double> tmp;
        tmp.resize(m);
        h2d(tmp.p, b, m, st);
        convert<double, T>(tmp.p, b0.p, m, st);
        MG_CK(cudaMemsetAsync(flags.p, 0, 8 * sizeof(int), st));
        pcg(iters, 0);
        convert<T, double>(xs.p, tmp.p, m, st);
        d2h(xo, tmp.p, m, st);
        MG_CK(cudaStreamSynchronize(st));
    }
};

}  // namespace mgpbd

// ============================================================================ C ABI
struct mgpbd_ctx {
    std::unique_ptr<mgpbd::EngineBase> eng;
    std::string err;
};

using mgpbd::Error;

template <class F>
static mgpbd_status guarded(mgpbd_ctx* ctx, F&& f) {
    if (!ctx) return MGPBD_E_ARG;
    try {
        ctx->eng->bind();
        f();
        return MGPBD_OK;
    } catch (const Error& e) {
        ctx->err = e.what();
        return (mgpbd_status)e.status;
    } catch (const std::exception& e) {
        ctx->err = e.what();
        return MGPBD_E_CUDA;
    }
}

extern "C" {

mgpbd_status mgpbd_config_default(mgpbd_config* c) {
    if (!c) return MGPBD_E_ARG;
    std::memset(c, 0, sizeof(*c));
    c->precision = 0;
    c->theta = 0.1;
    c->k_nullspace = 1;
    c->min_coarse = 400;
    c->max_levels = 16;
    c->stall_ratio = 0.9;
    c->setup_interval = 20;
    c->bootstrap_sweeps = 20;
    c->power_iters = 100;
    c->lambda_min_est = 0.1;
    c->lambda_safety = 1.1;
    c->smoother_sweeps = 2;
    c->pcg_iters = 10;
    c->omega_relax = 0.1;
    c->gravity[0] = 0.0; c->gravity[1] = -9.8; c->gravity[2] = 0.0;
    c->seed = 1;
    c->device = 0;
    c->stream = nullptr;
    c->max_dense_coarse = 2048;
    c->rank = 0; c->world = 1;
    c->profile = 0;
    c->nccl_id = nullptr;
    c->vgroup = nullptr;
    c->level0_operator = 1;
    c->smoother = 0;
    c->cheb_lower = 0.25;
    c->backtrack = 0;
    c->omega_min = 1e-3;
    c->residual_tol = 0.0;
    c->pcg_tol = 0.0;
    c->residual_abs = 0.0;
    c->resetup_on_indef = 1;
    c->omega_refresh_iters = 0;
    c->time_budget_ms = 0.0;
    return MGPBD_OK;
}

static std::string g_create_err;

mgpbd_status mgpbd_create(const mgpbd_mesh* mesh, const mgpbd_constraints* cons, const double* inv_mass,
                          const double* compliance, const mgpbd_config* cfg, mgpbd_ctx** out) {
    if (!out) return MGPBD_E_ARG;
    *out = nullptr;
    auto fail = [&](const std::string& m) { g_create_err = m; return MGPBD_E_ARG; };
    if (!mesh || !cons || !inv_mass || !compliance || !cfg) return fail("NULL argument");
    if (!mesh->rest_pos || mesh->n_verts <= 0) return fail("bad mesh");
    if (cons->kind != MGPBD_DISTANCE && cons->kind != MGPBD_TET_ARAP) return fail("bad constraint kind");
    if (cons->n_cons <= 0 || !cons->verts) return fail("bad constraint set");
    if ((int64_t)cons->n_cons * cons->kind >= ((int64_t)1 << 31)) return fail("too many constraints");
    if (cfg->precision != 0 && cfg->precision != 1) return fail("precision must be 0 (fp64) or 1 (fp32)");
    if (cfg->k_nullspace < 1 || cfg->k_nullspace > 8) return fail("k_nullspace must be in 1..8 (reading c1; f2)");
    if (cfg->k_nullspace > 1 && (cfg->world > 1 || cfg->vgroup || cfg->nccl_id))
        return fail("k_nullspace > 1 runs on one rank");
    if (cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world) return fail("bad rank/world");
    if (cfg->world > 1 && !cfg->nccl_id && !cfg->vgroup) return fail("world > 1 needs nccl_id or vgroup");
    if (cfg->level0_operator != 0 && cfg->level0_operator != 1) return fail("level0_operator must be 0 or 1");
    if (cfg->smoother < 0 || cfg->smoother > 2)
        return fail("smoother must be 0 (omega-Jacobi), 1 (Chebyshev) or 2 (multicolour Gauss-Seidel)");
    if (cfg->smoother == 2 && (cfg->level0_operator != 0 || cfg->world > 1 || cfg->vgroup || cfg->nccl_id))
        return fail("the Gauss-Seidel smoother needs level0_operator = 0 and one rank");
    if (cfg->smoother_sweeps > 8) return fail("smoother_sweeps must be <= 8");
    if (cfg->backtrack != 0 && cfg->backtrack != 1) return fail("backtrack must be 0 or 1");
    if (!(cfg->omega_min > 0.0) || !(cfg->residual_tol >= 0.0) || !(cfg->residual_abs >= 0.0))
        return fail("bad omega_min / residual_tol / residual_abs");
    if (cfg->smoother == 1 && !(cfg->cheb_lower > 0.0 && cfg->cheb_lower < 1.0)) return fail("cheb_lower must be in (0, 1)");
    if (!(cfg->pcg_tol >= 0.0)) return fail("pcg_tol must be >= 0");
    if (cfg->omega_refresh_iters < 0 || cfg->omega_refresh_iters > 10000) return fail("omega_refresh_iters must be in 0..10000");
    if (!(cfg->time_budget_ms >= 0.0)) return fail("time_budget_ms must be >= 0");
    if (cfg->smoother_sweeps < 1 || cfg->pcg_iters < 0 || cfg->pcg_iters > mgpbd::SC_KMAX || cfg->setup_interval < 1 ||
        cfg->min_coarse < 1 || cfg->max_levels < 1 || cfg->power_iters < 0 || cfg->bootstrap_sweeps < 0 ||
        cfg->max_dense_coarse < 1)
        return fail("bad config");
    const int kc = cons->kind;
    for (int64_t j = 0; j < cons->n_cons; ++j) {
        for (int a = 0; a < kc; ++a) {
            int32_t va = cons->verts[j * kc + a];
            if (va < 0 || va >= mesh->n_verts) return fail("vertex id out of range in constraint " + std::to_string(j));
            for (int b = a + 1; b < kc; ++b)
                if (cons->verts[j * kc + b] == va) return fail("repeated vertex in constraint " + std::to_string(j));
        }
        if (!(compliance[j] >= 0.0)) return fail("negative compliance");
    }
    for (int32_t i = 0; i < mesh->n_verts; ++i)
        if (!(inv_mass[i] >= 0.0)) return fail("negative inverse mass");
    auto* ctx = new mgpbd_ctx();
    try {
        if (cfg->precision == 1) ctx->eng.reset(new mgpbd::Engine<float>(mesh, cons, inv_mass, compliance, cfg));
        else ctx->eng.reset(new mgpbd::Engine<double>(mesh, cons, inv_mass, compliance, cfg));
    } catch (const Error& e) {
        g_create_err = e.what();
        delete ctx;
        return (mgpbd_status)e.status;
    } catch (const std::exception& e) {
        g_create_err = e.what();
        delete ctx;
        return MGPBD_E_CUDA;
    }
    *out = ctx;
    return MGPBD_OK;
}

mgpbd_status mgpbd_setup_hierarchy(mgpbd_ctx* ctx) {
    return guarded(ctx, [&] { ctx->eng->stale = true; });
}

mgpbd_status mgpbd_step(mgpbd_ctx* ctx, double dt, int32_t n_iters) {
    if (ctx && (!(dt > 0.0) || n_iters < 1 || n_iters > MGPBD_MAX_FRAME_ITERS)) {
        ctx->err = "dt must be > 0 and 1 <= n_iters <= MGPBD_MAX_FRAME_ITERS";
        return MGPBD_E_ARG;
    }
    return guarded(ctx, [&] { ctx->eng->step(dt, n_iters); });
}

mgpbd_status mgpbd_set_profiling(mgpbd_ctx* ctx, int32_t on) {
    return guarded(ctx, [&] { ctx->eng->set_profiling(on); });
}

mgpbd_status mgpbd_set_state(mgpbd_ctx* ctx, const double* pos, const double* vel) {
    return guarded(ctx, [&] { ctx->eng->set_state(pos, vel); });
}
mgpbd_status mgpbd_get_positions(mgpbd_ctx* ctx, double* out) {
    if (ctx && !out) return MGPBD_E_ARG;
    return guarded(ctx, [&] { ctx->eng->get_positions(out); });
}
mgpbd_status mgpbd_get_velocities(mgpbd_ctx* ctx, double* out) {
    if (ctx && !out) return MGPBD_E_ARG;
    return guarded(ctx, [&] { ctx->eng->get_velocities(out); });
}
mgpbd_status mgpbd_get_lambda(mgpbd_ctx* ctx, double* out) {
    if (ctx && !out) return MGPBD_E_ARG;
    return guarded(ctx, [&] { ctx->eng->get_lambda(out); });
}
mgpbd_status mgpbd_get_stats(mgpbd_ctx* ctx, mgpbd_stats* out) {
    if (ctx && !out) return MGPBD_E_ARG;
    return guarded(ctx, [&] { ctx->eng->get_stats(out); });
}
mgpbd_status mgpbd_get_level_sizes(mgpbd_ctx* ctx, int32_t l, int64_t* n, int64_t* nnz) {
    if (ctx && (!n || !nnz)) return MGPBD_E_ARG;
    return guarded(ctx, [&] { ctx->eng->level_sizes(l, n, nnz); });
}
mgpbd_status mgpbd_get_level(mgpbd_ctx* ctx, int32_t l, int64_t* rowptr, int32_t* cols, double* vals) {
    return guarded(ctx, [&] { ctx->eng->get_level(l, rowptr, cols, vals); });
}
mgpbd_status mgpbd_get_prolongator_csr(mgpbd_ctx* ctx, int32_t l, int64_t* nnz, int64_t* rowptr, int32_t* col,
                                       double* val) {
    if (!nnz) return MGPBD_E_ARG;
    return guarded(ctx, [&] { ctx->eng->get_prolongator_csr(l, nnz, rowptr, col, val); });
}
mgpbd_status mgpbd_get_prolongator(mgpbd_ctx* ctx, int32_t l, double* p) {
    if (ctx && !p) return MGPBD_E_ARG;
    return guarded(ctx, [&] { ctx->eng->get_prolongator(l, p); });
}
mgpbd_status mgpbd_get_aggregates(mgpbd_ctx* ctx, int32_t l, int32_t* out) {
    if (ctx && !out) return MGPBD_E_ARG;
    return guarded(ctx, [&] { ctx->eng->get_aggregates(l, out); });
}
mgpbd_status mgpbd_get_near_kernel(mgpbd_ctx* ctx, double* out) {
    if (ctx && !out) return MGPBD_E_ARG;
    return guarded(ctx, [&] { ctx->eng->get_near_kernel(out); });
}
mgpbd_status mgpbd_debug_setup_from(mgpbd_ctx* ctx, const double* vals) {
    if (ctx && !vals) return MGPBD_E_ARG;
    return guarded(ctx, [&] { ctx->eng->debug_setup_from(vals); });
}
mgpbd_status mgpbd_debug_vcycle(mgpbd_ctx* ctx, const double* b, double* x) {
    if (ctx && (!b || !x)) return MGPBD_E_ARG;
    return guarded(ctx, [&] { ctx->eng->debug_vcycle(b, x); });
}
mgpbd_status mgpbd_debug_prepare(mgpbd_ctx* ctx, double dt) {
    if (!ctx || !(dt > 0.0)) return MGPBD_E_ARG;
    return guarded(ctx, [&] { ctx->eng->debug_prepare(dt); });
}
mgpbd_status mgpbd_debug_pcg(mgpbd_ctx* ctx, const double* b, int32_t iters, double* x) {
    if (ctx && (!b || !x || iters < 0 || iters > mgpbd::SC_KMAX)) return MGPBD_E_ARG;
    return guarded(ctx, [&] { ctx->eng->debug_pcg(b, iters, x); });
}
mgpbd_status mgpbd_pass_burst(mgpbd_ctx* ctx, int32_t reps, double* ms, double* bytes) {
    if (ctx && (reps < 1 || reps > 4096 || !ms || !bytes)) return MGPBD_E_ARG;
    return guarded(ctx, [&] { ctx->eng->pass_burst(reps, ms, bytes); });
}
mgpbd_status mgpbd_nccl_unique_id(void* out128) {
    if (!out128) return MGPBD_E_ARG;
    try {
        mgpbd::nccl_unique_id(out128);
    } catch (const Error& e) {
        g_create_err = e.what();
        return (mgpbd_status)e.status;
    }
    return MGPBD_OK;
}
mgpbd_status mgpbd_vgroup_create(int32_t world, void** out) {
    if (!out || world < 1 || world > 8) return MGPBD_E_ARG;
    *out = mgpbd::vgroup_create(world);
    return MGPBD_OK;
}
void mgpbd_vgroup_destroy(void* g) { mgpbd::vgroup_destroy(static_cast<mgpbd::VirtualGroup*>(g)); }
mgpbd_status mgpbd_partition_rows(const int64_t* rowptr, int32_t n, int32_t world, int32_t* bounds) {
    if (!rowptr || !bounds || n < 0 || world < 1) return MGPBD_E_ARG;
    const std::vector<int32_t> b = mgpbd::partition_rows(rowptr, n, world);
    std::memcpy(bounds, b.data(), sizeof(int32_t) * b.size());
    return MGPBD_OK;
}
mgpbd_status mgpbd_halo_plan(const int32_t* bounds, const int32_t* minc, const int32_t* maxc, int32_t world,
                             int32_t* recv) {
    if (!bounds || !minc || !maxc || !recv || world < 1) return MGPBD_E_ARG;
    std::vector<int32_t> b(bounds, bounds + world + 1), mn(minc, minc + world), mx(maxc, maxc + world);
    const auto plan = mgpbd::halo_plan(b, mn, mx);
    for (int q = 0; q < world; ++q)
        for (int p = 0; p < world; ++p) {
            recv[(q * world + p) * 2] = plan[q][p].a;
            recv[(q * world + p) * 2 + 1] = plan[q][p].b;
        }
    return MGPBD_OK;
}

const char* mgpbd_last_error(const mgpbd_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }
void mgpbd_destroy(mgpbd_ctx* ctx) {
    if (!ctx) return;
    if (ctx->eng) ctx->eng->bind();
    delete ctx;
}

}  // extern "C"
