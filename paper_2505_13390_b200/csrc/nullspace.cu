// k > 1 near-kernel setup and transfer kernels, see nullspace.cuh.
#include <algorithm>
#include <cstdint>
#include <vector>

#include "nullspace.cuh"
#include "util.cuh"

namespace mgpbd {

namespace {

constexpr int KMAX = 8;

// one thread per item (the kernels below are not grid-stride): the grid must cover every item — a cap here left
// items beyond 148 x 64 x 256 uncomputed (k = 6 on blockslab32 and larger: garbage block Galerkin values)
inline int g1(int64_t n, int bs = 256) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + bs - 1) / bs, INT32_MAX)); }

// Warp per aggregate: MGS thin QR of the |N_a| x k block (members in mlist order = ascending node index),
// one re-orthogonalisation pass, drop test |v_perp| <= tol |B_a[:,c]| (reading c24), zero block -> uniform
// column (reading c25).  Q goes to Qs[(slot) k + j], R (k x k, row j = kept column j) to Rt[a k k + j k + c].
__global__ void k_qr(int32_t n, int32_t n_agg, int k, const int64_t* __restrict__ mptr,
                     const int32_t* __restrict__ mlist, const double* __restrict__ B, double tol,
                     double* __restrict__ Qs, int32_t* __restrict__ rk, double* __restrict__ Rt) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t a = w0; a < n_agg; a += nw) {
        const int64_t m0 = mptr[a];
        const int32_t na = (int32_t)(mptr[a + 1] - m0);
        double R[KMAX * KMAX];
#pragma unroll
        for (int q = 0; q < KMAX * KMAX; ++q) R[q] = 0.0;
        int r = 0;
        for (int c = 0; c < k; ++c) {
            double bn = 0.0;
            for (int32_t t = lane; t < na; t += 32) {
                const double v = B[(int64_t)c * n + mlist[m0 + t]];
                Qs[(m0 + t) * k + r] = v;
                bn += v * v;
            }
            bn = sqrt(group_sum<32>(bn));
            for (int pass = 0; pass < 2; ++pass)
                for (int j = 0; j < r; ++j) {
                    double s = 0.0;
                    for (int32_t t = lane; t < na; t += 32) s += Qs[(m0 + t) * k + j] * Qs[(m0 + t) * k + r];
                    s = group_sum<32>(s);
                    for (int32_t t = lane; t < na; t += 32) Qs[(m0 + t) * k + r] -= s * Qs[(m0 + t) * k + j];
                    R[j * KMAX + c] += s;
                }
            double vn = 0.0;
            for (int32_t t = lane; t < na; t += 32) { const double v = Qs[(m0 + t) * k + r]; vn += v * v; }
            vn = sqrt(group_sum<32>(vn));
            if (vn > 0.0 && vn > tol * bn) {
                for (int32_t t = lane; t < na; t += 32) Qs[(m0 + t) * k + r] = Qs[(m0 + t) * k + r] / vn;
                R[r * KMAX + c] = vn;
                ++r;
            }
        }
        if (r == 0) {
            const double u = 1.0 / sqrt((double)na);
            for (int32_t t = lane; t < na; t += 32) Qs[(m0 + t) * k] = u;
            for (int c = 0; c < KMAX; ++c) R[c] = 0.0;
            r = 1;
        }
        if (lane == 0) {
            rk[a] = r;
            for (int j = 0; j < k; ++j)
                for (int c = 0; c < k; ++c) Rt[(a * k + j) * k + c] = j < r ? R[j * KMAX + c] : 0.0;
        }
    }
}

__global__ void k_i64_to_i32(int64_t n, const int64_t* __restrict__ in, int32_t* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = (int32_t)in[i];
}

__global__ void k_qr_out(int32_t n_agg, int k, const int32_t* __restrict__ rk, const int32_t* __restrict__ coff,
                         const double* __restrict__ Rt, int32_t nc, double* __restrict__ Bn, int32_t* __restrict__ dof_agg) {
    const int32_t a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= n_agg) return;
    for (int j = 0; j < rk[a]; ++j) {
        dof_agg[coff[a] + j] = a;
        for (int c = 0; c < k; ++c) Bn[(int64_t)c * nc + coff[a] + j] = Rt[((int64_t)a * k + j) * k + c];
    }
}

__global__ void k_rowlen_from_agg(int32_t n, const int32_t* __restrict__ agg, const int32_t* __restrict__ rk,
                                  int32_t* __restrict__ len) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) len[i] = rk[agg[i]];
}

__global__ void k_p_fill(int32_t n, int k, const int32_t* __restrict__ mlist, const int32_t* __restrict__ agg,
                         const int32_t* __restrict__ rk, const int32_t* __restrict__ coff, const double* __restrict__ Qs,
                         const int64_t* __restrict__ pptr, int32_t* __restrict__ pcol, double* __restrict__ pval) {
    const int64_t slot = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (slot >= n) return;
    const int32_t i = mlist[slot], a = agg[i];
    for (int j = 0; j < rk[a]; ++j) {
        pcol[pptr[i] + j] = coff[a] + j;
        pval[pptr[i] + j] = Qs[slot * k + j];
    }
}

// row length of aggregate row a in DOFs: sum of r_b over its entries; xoff per entry (ascending-column
// prefix of r over the row's entries, the diagonal entry at its sorted place)
__global__ void k_xrow_agg(int32_t n_agg, const int64_t* __restrict__ arow, const int32_t* __restrict__ acol,
                           const int32_t* __restrict__ coff, int32_t* __restrict__ alen, int64_t* __restrict__ xoff) {
    const int32_t a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= n_agg) return;
    const int64_t e0 = arow[a], e1 = arow[a + 1];   // off-diagonals ascending, diagonal (a) at e1 - 1
    const int32_t ra = coff[a + 1] - coff[a];
    int64_t cum = 0;
    bool diag_done = false;
    for (int64_t e = e0; e < e1 - 1; ++e) {
        const int32_t b = acol[e];
        if (!diag_done && b > a) { xoff[e1 - 1] = cum; cum += ra; diag_done = true; }
        xoff[e] = cum;
        cum += coff[b + 1] - coff[b];
    }
    if (!diag_done) { xoff[e1 - 1] = cum; cum += ra; }
    alen[a] = (int32_t)cum;
}

__global__ void k_xrow_len(int32_t nc, const int32_t* __restrict__ dof_agg, const int32_t* __restrict__ alen,
                           int32_t* __restrict__ len) {
    const int32_t I = blockIdx.x * blockDim.x + threadIdx.x;
    if (I < nc) len[I] = alen[dof_agg[I]];
}

// expanded columns of DOF row I = (a, c): blocks in ascending column order without (a, c), then (a, c)
__global__ void k_xcol(int32_t nc, const int32_t* __restrict__ dof_agg, const int32_t* __restrict__ coff,
                       const int64_t* __restrict__ arow, const int32_t* __restrict__ acol,
                       const int64_t* __restrict__ xrow, int32_t* __restrict__ xcol) {
    const int32_t I = blockIdx.x * blockDim.x + threadIdx.x;
    if (I >= nc) return;
    const int32_t a = dof_agg[I];
    const int64_t e0 = arow[a], e1 = arow[a + 1];
    int64_t p = xrow[I];
    auto block = [&](int32_t b) {
        for (int32_t J = coff[b]; J < coff[b + 1]; ++J)
            if (J != I) xcol[p++] = J;
    };
    bool diag_done = false;
    for (int64_t e = e0; e < e1 - 1; ++e) {
        const int32_t b = acol[e];
        if (!diag_done && b > a) { block(a); diag_done = true; }
        block(b);
    }
    if (!diag_done) block(a);
    xcol[p] = I;
}

// stage 1: W_t[d] = sum_{e in segment t} A_e P_{col(e), d}
template <class T>
__global__ void k_kgal1(int64_t T_, int k, const int64_t* __restrict__ tstart, const int32_t* __restrict__ trow,
                        const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                        const uint16_t* __restrict__ gperm, const T* __restrict__ val, const int64_t* __restrict__ pptr,
                        const T* __restrict__ pval, T* __restrict__ W) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= T_) return;
    const int32_t i = trow[t];
    const int64_t e0 = rowptr[i];
    double s[KMAX];
#pragma unroll
    for (int d = 0; d < KMAX; ++d) s[d] = 0.0;
    int rb = 0;
    for (int64_t q = tstart[t]; q < tstart[t + 1]; ++q) {
        const int64_t e = e0 + gperm[q];
        const int32_t j = col[e];
        const int64_t p0 = pptr[j];
        rb = (int)(pptr[j + 1] - p0);
        const double a = (double)val[e];
#pragma unroll
        for (int d = 0; d < KMAX; ++d)
            if (d < rb) s[d] += a * (double)pval[p0 + d];
    }
    for (int d = 0; d < k; ++d) W[t * k + d] = (T)(d < rb ? s[d] : 0.0);
}

// stage 2: thread per (aggregate entry E = (a, b), c < r_a): (A_c)_{(a,c),(b,d)} = sum_t P_{row(t),c} W_t[d]
template <class T>
__global__ void k_kgal2(int64_t annz, int k, const int64_t* __restrict__ lptr, const int32_t* __restrict__ llist,
                        const int32_t* __restrict__ trow, const T* __restrict__ W, const int64_t* __restrict__ pptr,
                        const T* __restrict__ pval, const int32_t* __restrict__ coff, const int32_t* __restrict__ erow,
                        const int32_t* __restrict__ acol, const int64_t* __restrict__ xoff,
                        const int64_t* __restrict__ xrow, T* __restrict__ cval) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (tid >= annz * k) return;
    const int64_t E = tid / k;
    const int c = (int)(tid % k);
    const int32_t a = erow[E], b = acol[E];
    const int ra = coff[a + 1] - coff[a], rb = coff[b + 1] - coff[b];
    if (c >= ra) return;
    double s[KMAX];
#pragma unroll
    for (int d = 0; d < KMAX; ++d) s[d] = 0.0;
    for (int64_t q = lptr[E]; q < lptr[E + 1]; ++q) {
        const int32_t t = llist[q];
        const double pc = (double)pval[pptr[trow[t]] + c];
#pragma unroll
        for (int d = 0; d < KMAX; ++d)
            if (d < rb) s[d] += pc * (double)W[(int64_t)t * k + d];
    }
    const int32_t I = coff[a] + c;
    const int64_t rs = xrow[I], re = xrow[I + 1];
    for (int d = 0; d < rb; ++d) {
        int64_t pos;
        if (b != a) pos = rs + xoff[E] + d - (b > a ? 1 : 0);
        else pos = d < c ? rs + xoff[E] + d : (d > c ? rs + xoff[E] + d - 1 : re - 1);
        cval[pos] = (T)s[d];
    }
}

__global__ void k_entry_row(int32_t n_agg, const int64_t* __restrict__ arow, int32_t* __restrict__ erow) {
    const int32_t a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= n_agg) return;
    for (int64_t e = arow[a]; e < arow[a + 1]; ++e) erow[e] = a;
}

template <class T>
__global__ void k_krestrict(int32_t nc, int k, const int32_t* __restrict__ dof_agg, const int32_t* __restrict__ coff,
                            const int64_t* __restrict__ mptr, const int32_t* __restrict__ mlist, const T* __restrict__ Qs,
                            const T* __restrict__ r, T* __restrict__ bc) {
    const int32_t J = blockIdx.x * blockDim.x + threadIdx.x;
    if (J >= nc) return;
    const int32_t a = dof_agg[J], j = J - coff[a];
    double s = 0.0;
    for (int64_t q = mptr[a]; q < mptr[a + 1]; ++q) s += (double)Qs[q * k + j] * (double)r[mlist[q]];
    bc[J] = (T)s;
}

template <class T>
__global__ void k_kprolong(int32_t row0, int32_t rows, const int64_t* __restrict__ pptr, const int32_t* __restrict__ pcol,
                           const T* __restrict__ pval, const T* __restrict__ e, T* __restrict__ x) {
    const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= rows) return;
    const int32_t i = row0 + t;
    double s = (double)x[i];
    for (int64_t q = pptr[i]; q < pptr[i + 1]; ++q) s += (double)pval[q] * (double)e[pcol[q]];
    x[i] = (T)s;
}

}  // namespace

int32_t qr_prolongator(int32_t n, int32_t n_agg, int k, const int32_t* agg, const int64_t* mptr, const int32_t* mlist,
                       const double* B, double rank_tol, KProlongator& P, DBuf<double>& B_next, cudaStream_t s) {
    if (k < 1 || k > KMAX) throw Error(-1, "k_nullspace must be in 1..8");
    P.k = k; P.n = n; P.n_agg = n_agg;
    P.Qs64.resize((size_t)n * k);
    DBuf<int32_t> rk, len;
    DBuf<double> Rt;
    rk.resize(n_agg); Rt.resize((size_t)n_agg * k * k);
    k_qr<<<g1((int64_t)n_agg * 32, 128), 128, 0, s>>>(n, n_agg, k, mptr, mlist, B, rank_tol, P.Qs64.p, rk.p, Rt.p);
    MG_LAUNCH_CHECK();
    DBuf<int64_t> coff64;
    coff64.resize((size_t)n_agg + 1);
    scan_exclusive<int32_t>(rk.p, coff64.p, n_agg, s);
    P.coff.resize((size_t)n_agg + 1);
    k_i64_to_i32<<<g1((int64_t)n_agg + 1), 256, 0, s>>>((int64_t)n_agg + 1, coff64.p, P.coff.p);
    MG_LAUNCH_CHECK();
    P.nc = (int32_t)read_scalar(coff64.p + n_agg, s);
    P.dof_agg.resize(P.nc);
    B_next.resize((size_t)P.nc * k);
    k_qr_out<<<g1(n_agg), 256, 0, s>>>(n_agg, k, rk.p, P.coff.p, Rt.p, P.nc, B_next.p, P.dof_agg.p);
    MG_LAUNCH_CHECK();
    len.resize(n);
    k_rowlen_from_agg<<<g1(n), 256, 0, s>>>(n, agg, rk.p, len.p);
    MG_LAUNCH_CHECK();
    P.pptr.resize((size_t)n + 1);
    scan_exclusive<int32_t>(len.p, P.pptr.p, n, s);
    const int64_t pn = read_scalar(P.pptr.p + n, s);
    P.pcol.resize(pn); P.pval64.resize(pn);
    k_p_fill<<<g1(n), 256, 0, s>>>(n, k, mlist, agg, rk.p, P.coff.p, P.Qs64.p, P.pptr.p, P.pcol.p, P.pval64.p);
    MG_LAUNCH_CHECK();
    return P.nc;
}

void kgal_expand(int32_t n_agg, const int64_t* arow, const int32_t* acol, const int32_t* coff, DBuf<int64_t>& xrow,
                 DBuf<int32_t>& xcol, DBuf<int64_t>& xoff, DBuf<int32_t>& erow, cudaStream_t s) {
    const int64_t annz = read_scalar(arow + n_agg, s);
    const int32_t nc = read_scalar(coff + n_agg, s);
    DBuf<int32_t> alen, len, dof;
    alen.resize(n_agg); xoff.resize(annz); erow.resize(std::max<int64_t>(annz, 1));
    k_entry_row<<<g1(n_agg), 256, 0, s>>>(n_agg, arow, erow.p);
    MG_LAUNCH_CHECK();
    k_xrow_agg<<<g1(n_agg), 256, 0, s>>>(n_agg, arow, acol, coff, alen.p, xoff.p);
    MG_LAUNCH_CHECK();
    // DOF -> aggregate from the offsets (same as KProlongator::dof_agg; recomputed to keep this stand-alone)
    dof.resize(nc);
    {
        std::vector<int32_t> hc((size_t)n_agg + 1), hd(nc);
        d2h(hc.data(), coff, (size_t)n_agg + 1, s);
        MG_CK(cudaStreamSynchronize(s));
        for (int32_t a = 0; a < n_agg; ++a)
            for (int32_t J = hc[a]; J < hc[a + 1]; ++J) hd[J] = a;
        h2d(dof.p, hd.data(), nc, s);
    }
    len.resize(nc);
    k_xrow_len<<<g1(nc), 256, 0, s>>>(nc, dof.p, alen.p, len.p);
    MG_LAUNCH_CHECK();
    xrow.resize((size_t)nc + 1);
    scan_exclusive<int32_t>(len.p, xrow.p, nc, s);
    const int64_t xnnz = read_scalar(xrow.p + nc, s);
    xcol.resize(xnnz);
    k_xcol<<<g1(nc), 256, 0, s>>>(nc, dof.p, coff, arow, acol, xrow.p, xcol.p);
    MG_LAUNCH_CHECK();
    MG_CK(cudaStreamSynchronize(s));
}

template <class T>
void kgal_numeric(const GalerkinPlan& plan, const int64_t* rowptr, const int32_t* col, const T* val, int k,
                  const int64_t* pptr, const T* pval, const int32_t* coff, const int32_t* agg, int32_t n_agg,
                  const int32_t* erow, const int32_t* acol, const int64_t* xoff, const int64_t* xrow, int32_t nc,
                  T* W, T* cval, T* cdinv, cudaStream_t s) {
    (void)agg; (void)n_agg;
    if (plan.T) {
        k_kgal1<T><<<g1(plan.T), 256, 0, s>>>(plan.T, k, plan.tstart.p, plan.trow.p, rowptr, col, plan.gperm.p, val,
                                              pptr, pval, W);
        MG_LAUNCH_CHECK();
    }
    const int64_t annz = plan.lptr.n ? (int64_t)plan.lptr.n - 1 : 0;
    if (annz) {
        k_kgal2<T><<<g1(annz * k), 256, 0, s>>>(annz, k, plan.lptr.p, plan.llist.p, plan.trow.p, W, pptr, pval, coff,
                                                 erow, acol, xoff, xrow, cval);
        MG_LAUNCH_CHECK();
    }
    if (cdinv) diag_inv<T>(nc, xrow, cval, cdinv, s);
}

template <class T>
void krestrict(int32_t nc, int k, const int32_t* dof_agg, const int32_t* coff, const int64_t* mptr, const int32_t* mlist,
               const T* Qs, const T* r, T* bc, cudaStream_t s) {
    if (!nc) return;
    k_krestrict<T><<<g1(nc), 256, 0, s>>>(nc, k, dof_agg, coff, mptr, mlist, Qs, r, bc);
    MG_LAUNCH_CHECK();
}

template <class T>
void kprolong(int32_t row0, int32_t rows, const int64_t* pptr, const int32_t* pcol, const T* pval, const T* e, T* x,
              cudaStream_t s) {
    if (rows <= 0) return;
    k_kprolong<T><<<g1(rows), 256, 0, s>>>(row0, rows, pptr, pcol, pval, e, x);
    MG_LAUNCH_CHECK();
}

#define MG_INST(T)                                                                                                   \
    template void kgal_numeric<T>(const GalerkinPlan&, const int64_t*, const int32_t*, const T*, int, const int64_t*,  \
                                  const T*, const int32_t*, const int32_t*, int32_t, const int32_t*, const int32_t*,   \
                                  const int64_t*, const int64_t*, int32_t, T*, T*, T*, cudaStream_t);                  \
    template void krestrict<T>(int32_t, int, const int32_t*, const int32_t*, const int64_t*, const int32_t*, const T*, \
                               const T*, T*, cudaStream_t);                                                            \
    template void kprolong<T>(int32_t, int32_t, const int64_t*, const int32_t*, const T*, const T*, T*, cudaStream_t);
MG_INST(float)
MG_INST(double)
#undef MG_INST

}  // namespace mgpbd
