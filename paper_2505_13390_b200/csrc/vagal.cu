// Level-0 -> level-1 Galerkin product from the scaled gradients, see vagal.cuh.
#include <algorithm>

#include "setup.cuh"
#include "util.cuh"
#include "vagal.cuh"

namespace mgpbd {

namespace {

template <class T>
struct alignas(4 * sizeof(T)) G4 {
    T x, y, z, w;
};

inline int g1(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 32)); }

// per vertex: incidences re-sorted by aggregate (stable: codes stay ascending inside an aggregate),
// number of distinct aggregates
__global__ void k_va_sort(int32_t nv, int kc, const int64_t* __restrict__ vptr, const int32_t* __restrict__ vlist,
                          const int32_t* __restrict__ agg, const int64_t* __restrict__ ppos,
                          int32_t* __restrict__ vlist2, int32_t* __restrict__ vpos, int32_t* __restrict__ pcnt) {
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
        const int64_t e0 = vptr[v], e1 = vptr[v + 1];
        // vpos: position of the incidence in the hot vertex-major copy (padded layout when ppos is given)
        for (int64_t e = e0; e < e1; ++e) {
            vlist2[e] = vlist[e];
            if (vpos) vpos[e] = (int32_t)(ppos ? ppos[v] + (e - e0) : e);
        }
        for (int64_t a = e0 + 1; a < e1; ++a) {
            const int32_t c = vlist2[a];
            const int32_t pa = vpos ? vpos[a] : 0;
            const int32_t ka = agg[c / kc];
            int64_t b = a - 1;
            while (b >= e0) {
                const int32_t cb = vlist2[b];
                if (agg[cb / kc] <= ka) break;
                vlist2[b + 1] = cb;
                if (vpos) vpos[b + 1] = vpos[b];
                --b;
            }
            vlist2[b + 1] = c;
            if (vpos) vpos[b + 1] = pa;
        }
        int32_t pc = 0, prev = -1;
        for (int64_t e = e0; e < e1; ++e) {
            const int32_t k = agg[vlist2[e] / kc];
            if (k != prev) { ++pc; prev = k; }
        }
        pcnt[v] = pc;
    }
}

// pair starts / aggregates, and k_v^2 products per vertex
__global__ void k_va_pairs(int32_t nv, int kc, const int64_t* __restrict__ vptr, const int32_t* __restrict__ vlist2,
                           const int32_t* __restrict__ agg, const int64_t* __restrict__ vpp,
                           int32_t* __restrict__ pstart, int32_t* __restrict__ pagg, int32_t* __restrict__ ccnt) {
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
        const int64_t e0 = vptr[v], e1 = vptr[v + 1];
        int64_t p = vpp[v];
        int32_t prev = -1;
        for (int64_t e = e0; e < e1; ++e) {
            const int32_t k = agg[vlist2[e] / kc];
            if (k != prev) { pstart[p] = (int32_t)e; pagg[p] = k; ++p; prev = k; }
        }
        const int32_t kv = (int32_t)(vpp[v + 1] - vpp[v]);
        ccnt[v] = kv * kv;
    }
}

// position of (a, b) in the coarse CSR (off-diagonals ascending, diagonal last); -1 if absent
__device__ __forceinline__ int64_t coarse_pos(const int64_t* __restrict__ crowptr, const int32_t* __restrict__ ccol,
                                              int32_t a, int32_t b) {
    const int64_t r0 = crowptr[a], r1 = crowptr[a + 1];
    if (a == b) return r1 - 1;
    int64_t lo = r0, hi = r1 - 1;  // off-diagonal range [r0, r1-1)
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (ccol[mid] < b) lo = mid + 1;
        else hi = mid;
    }
    return (lo < r1 - 1 && ccol[lo] == b) ? lo : -1;
}

__global__ void k_va_contrib(int32_t nv, const int64_t* __restrict__ vpp, const int64_t* __restrict__ coff,
                             const int32_t* __restrict__ pagg, const int64_t* __restrict__ crowptr,
                             const int32_t* __restrict__ ccol, int32_t* __restrict__ key, int2* __restrict__ pq,
                             int32_t* __restrict__ bad) {
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
        const int64_t p0 = vpp[v], p1 = vpp[v + 1];
        int64_t idx = coff[v];
        for (int64_t p = p0; p < p1; ++p)
            for (int64_t q = p0; q < p1; ++q, ++idx) {
                const int64_t pos = coarse_pos(crowptr, ccol, pagg[p], pagg[q]);
                if (pos < 0) { atomicExch(bad, 1); key[idx] = 0; }
                else key[idx] = (int32_t)pos;
                pq[idx] = make_int2((int32_t)p, (int32_t)q);
            }
    }
}

__global__ void k_va_permute(int64_t n, const int32_t* __restrict__ list, const int2* __restrict__ in,
                             int2* __restrict__ out) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        out[k] = in[list[k]];
}

// product range of every off-diagonal entry; empty for the diagonal (k_va_a1_diag computes it)
__global__ void k_va_crange(int32_t n, const int64_t* __restrict__ crowptr, const int64_t* __restrict__ cptr,
                            int2* __restrict__ crange) {
    for (int32_t a = blockIdx.x * blockDim.x + threadIdx.x; a < n; a += gridDim.x * blockDim.x) {
        const int64_t k1 = crowptr[a + 1] - 1;
        for (int64_t k = crowptr[a]; k < k1; ++k) crange[k] = make_int2((int32_t)cptr[k], (int32_t)cptr[k + 1]);
        crange[k1] = make_int2(0, 0);
    }
}

// G_p = sum over the pair's incidences of P_j h_{j,s} (fp64 sum, incidence order)
// (HV: h read from the vertex-major copy hv of the matrix-free operator — the pair's incidences are
// neighbours there, instead of one 12-byte record per constraint scattered over h)
template <class T, int KC, bool HV>
__global__ void k_va_g(int64_t npairs, const int32_t* __restrict__ pstart, const int32_t* __restrict__ vlist2,
                       const int32_t* __restrict__ vpos, const T* __restrict__ h, const T* __restrict__ hv,
                       int64_t ninc, const T* __restrict__ P, G4<T>* __restrict__ G) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npairs; p += (int64_t)gridDim.x * blockDim.x) {
        double g0 = 0.0, g1_ = 0.0, g2 = 0.0;
        const int32_t e0 = pstart[p], e1 = pstart[p + 1];
        // chunks of 4 incidences: all index loads, then all P / h gathers, then the sums (in order)
        for (int32_t eb = e0; eb < e1; eb += 4) {
            int32_t code[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) code[q] = eb + q < e1 ? vlist2[eb + q] : -1;
            double pj[4], hx[4], hy[4], hz[4];
            if (HV) {
                int32_t pos[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) pos[q] = eb + q < e1 ? vpos[eb + q] : 0;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const bool in = code[q] >= 0;
                    pj[q] = in ? (double)P[code[q] / KC] : 0.0;
                    hx[q] = in ? (double)hv[pos[q]] : 0.0;
                    hy[q] = in ? (double)hv[ninc + pos[q]] : 0.0;
                    hz[q] = in ? (double)hv[2 * ninc + pos[q]] : 0.0;
                }
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const bool in = code[q] >= 0;
                    const T* hh = h + (int64_t)(in ? code[q] : 0) * 3;
                    pj[q] = in ? (double)P[code[q] / KC] : 0.0;
                    hx[q] = in ? (double)hh[0] : 0.0;
                    hy[q] = in ? (double)hh[1] : 0.0;
                    hz[q] = in ? (double)hh[2] : 0.0;
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                g0 += pj[q] * hx[q];
                g1_ += pj[q] * hy[q];
                g2 += pj[q] * hz[q];
            }
        }
        G[p] = G4<T>{(T)g0, (T)g1_, (T)g2, (T)0};
    }
}

// Off-diagonal entries (A_1)_ab: one thread each over the entry's product range (chunks of 4: all
// (p, q) loads, then all G gathers, then the sums in order).
template <class T>
__global__ void k_va_a1(int64_t cnnz, const int2* __restrict__ crange, const int2* __restrict__ cpq,
                        const G4<T>* __restrict__ G, T* __restrict__ cval) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < cnnz; k += (int64_t)gridDim.x * blockDim.x) {
        const int2 rg = crange[k];
        if (rg.x == rg.y) continue;  // diagonal: k_va_a1_diag
        double s = 0.0;
        for (int32_t cb = rg.x; cb < rg.y; cb += 4) {
            int2 pq[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) pq[u] = cb + u < rg.y ? cpq[cb + u] : make_int2(-1, -1);
            G4<T> a[4], b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const bool in = pq[u].x >= 0;
                a[u] = in ? G[pq[u].x] : G4<T>{(T)0, (T)0, (T)0, (T)0};
                b[u] = in ? G[pq[u].y] : G4<T>{(T)0, (T)0, (T)0, (T)0};
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                s += (double)a[u].x * (double)b[u].x + (double)a[u].y * (double)b[u].y + (double)a[u].z * (double)b[u].z;
        }
        cval[k] = (T)s;
    }
}

// Diagonal entries (A_1)_aa: one warp per aggregate (the diagonal collects a product from every vertex
// the aggregate touches, ~10-50x the work of an off-diagonal entry; thread-per-entry left whole warps
// waiting on it).  Lane-strided chunks of 4 products + the aggregate's sum_i P_i^2 at_i, fixed-order
// butterfly (deterministic); writes the smoother's 1/(A_1)_aa as well.
template <class T>
__global__ void k_va_a1_diag(int32_t n_agg, const int64_t* __restrict__ cptr, const int2* __restrict__ cpq,
                             const G4<T>* __restrict__ G, const int64_t* __restrict__ crowptr,
                             const int64_t* __restrict__ mptr, const int32_t* __restrict__ mlist,
                             const T* __restrict__ P, const T* __restrict__ at, T* __restrict__ cval,
                             T* __restrict__ cdinv) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t a = gw; a < n_agg; a += nw) {
        const int64_t k = crowptr[a + 1] - 1;
        const int64_t c0 = cptr[k], c1 = cptr[k + 1];
        double s = 0.0;
        for (int64_t cb = c0 + lane; cb < c1; cb += 4 * 32) {
            int2 pq[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) pq[u] = cb + 32 * u < c1 ? cpq[cb + 32 * u] : make_int2(-1, -1);
            G4<T> x[4], y[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const bool in = pq[u].x >= 0;
                x[u] = in ? G[pq[u].x] : G4<T>{(T)0, (T)0, (T)0, (T)0};
                y[u] = in ? G[pq[u].y] : G4<T>{(T)0, (T)0, (T)0, (T)0};
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                s += (double)x[u].x * (double)y[u].x + (double)x[u].y * (double)y[u].y + (double)x[u].z * (double)y[u].z;
        }
        for (int64_t e = mptr[a] + lane; e < mptr[a + 1]; e += 32) {  // sum_{i in a} P_i^2 at_i
            const int32_t i = mlist[e];
            const double pi = (double)P[i];
            s += pi * pi * (double)at[i];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
            const T d = (T)s;
            cval[k] = d;
            cdinv[a] = (T)(1.0 / (double)d);
        }
    }
}

__global__ void k_pat_count(int32_t nv, const int64_t* __restrict__ vpp, const int32_t* __restrict__ pagg,
                            int32_t* __restrict__ cnt) {
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
        const int64_t p0 = vpp[v], p1 = vpp[v + 1];
        const int32_t kv = (int32_t)(p1 - p0);
        for (int64_t p = p0; p < p1; ++p) atomicAdd(&cnt[pagg[p]], kv);
    }
}
// candidates of row a: every b that shares a vertex with a (order within a row fixed later by a sort)
__global__ void k_pat_fill(int32_t nv, const int64_t* __restrict__ vpp, const int32_t* __restrict__ pagg,
                           const int64_t* __restrict__ ptr, int32_t* __restrict__ cur, int32_t* __restrict__ cand) {
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
        const int64_t p0 = vpp[v], p1 = vpp[v + 1];
        const int32_t kv = (int32_t)(p1 - p0);
        for (int64_t p = p0; p < p1; ++p) {
            const int32_t a = pagg[p];
            const int64_t base = ptr[a] + atomicAdd(&cur[a], kv);
            for (int64_t q = p0; q < p1; ++q) cand[base + (q - p0)] = pagg[q];
        }
    }
}
// per row: unique sorted candidates except a, then a (diagonal last); count pass (out == nullptr) or fill
__global__ void k_pat_unique(int32_t n, const int64_t* __restrict__ ptr, const int32_t* __restrict__ cand,
                             int32_t* __restrict__ ucnt, const int64_t* __restrict__ crowptr, int32_t* __restrict__ out) {
    for (int32_t a = blockIdx.x * blockDim.x + threadIdx.x; a < n; a += gridDim.x * blockDim.x) {
        int64_t o = out ? crowptr[a] : 0;
        int32_t u = 0, prev = -1;
        for (int64_t k = ptr[a]; k < ptr[a + 1]; ++k) {
            const int32_t b = cand[k];
            if (b == prev || b == a) { prev = b; continue; }
            prev = b;
            if (out) out[o++] = b;
            ++u;
        }
        if (out) out[o] = a;
        else ucnt[a] = u + 1;
    }
}
__global__ void k_va_at(int32_t m, const double* __restrict__ alpha, double dt2, double* __restrict__ at) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) at[i] = alpha[i] / dt2;
}

}  // namespace

void va_coarse_pattern(int32_t nv, int kc, const int64_t* vptr, const int32_t* vlist, const int32_t* agg,
                       int32_t n_agg, DBuf<int64_t>& crowptr, DBuf<int32_t>& ccol, cudaStream_t s) {
    const int64_t ninc = read_scalar(vptr + nv, s);
    DBuf<int32_t> vl2, pcnt, pst, pagg, ccnt, cnt, cur, cand, ucnt;
    DBuf<int64_t> vpp, ptr;
    vl2.resize(ninc);
    pcnt.resize(nv);
    k_va_sort<<<g1(nv), 256, 0, s>>>(nv, kc, vptr, vlist, agg, nullptr, vl2.p, nullptr, pcnt.p);
    MG_LAUNCH_CHECK();
    vpp.resize((size_t)nv + 1);
    scan_exclusive<int32_t>(pcnt.p, vpp.p, nv, s);
    const int64_t npairs = read_scalar(vpp.p + nv, s);
    pst.resize(npairs + 1); pagg.resize(npairs); ccnt.resize(nv);
    k_va_pairs<<<g1(nv), 256, 0, s>>>(nv, kc, vptr, vl2.p, agg, vpp.p, pst.p, pagg.p, ccnt.p);
    MG_LAUNCH_CHECK();
    cnt.resize(n_agg);
    MG_CK(cudaMemsetAsync(cnt.p, 0, sizeof(int32_t) * (size_t)n_agg, s));
    k_pat_count<<<g1(nv), 256, 0, s>>>(nv, vpp.p, pagg.p, cnt.p);
    MG_LAUNCH_CHECK();
    ptr.resize((size_t)n_agg + 1);
    scan_exclusive<int32_t>(cnt.p, ptr.p, n_agg, s);
    const int64_t ncand = read_scalar(ptr.p + n_agg, s);
    cand.resize(ncand);
    cur.resize(n_agg);
    MG_CK(cudaMemsetAsync(cur.p, 0, sizeof(int32_t) * (size_t)n_agg, s));
    k_pat_fill<<<g1(nv), 256, 0, s>>>(nv, vpp.p, pagg.p, ptr.p, cur.p, cand.p);
    MG_LAUNCH_CHECK();
    sort_segments_i32(ptr.p, cand.p, n_agg, s);
    ucnt.resize(n_agg);
    k_pat_unique<<<g1(n_agg), 256, 0, s>>>(n_agg, ptr.p, cand.p, ucnt.p, nullptr, nullptr);
    MG_LAUNCH_CHECK();
    crowptr.resize((size_t)n_agg + 1);
    scan_exclusive<int32_t>(ucnt.p, crowptr.p, n_agg, s);
    ccol.resize(read_scalar(crowptr.p + n_agg, s));
    k_pat_unique<<<g1(n_agg), 256, 0, s>>>(n_agg, ptr.p, cand.p, nullptr, crowptr.p, ccol.p);
    MG_LAUNCH_CHECK();
    MG_CK(cudaStreamSynchronize(s));  // temporaries are freed on return
}

void va_at(int32_t m, const double* alpha, double dt, double* at, cudaStream_t s) {
    if (!m) return;
    k_va_at<<<g1(m), 256, 0, s>>>(m, alpha, dt * dt, at);
    MG_LAUNCH_CHECK();
}

void va_symbolic(int32_t nv, int kc, const int64_t* vptr, const int32_t* vlist, const int32_t* agg, int32_t n_agg,
                 const int64_t* crowptr, const int32_t* ccol, int64_t cnnz, VaPlan& plan, cudaStream_t s,
                 const int64_t* ppos, int64_t hv_stride) {
    const int64_t ninc = read_scalar(vptr + nv, s);
    plan.hv_stride = ppos ? hv_stride : ninc;
    plan.cnnz = cnnz;
    plan.vlist2.resize(ninc);
    plan.vpos.resize(ninc);
    plan.ninc = ninc;
    DBuf<int32_t> pcnt, pagg, ccnt, key, clist, cnt;
    DBuf<int64_t> vpp, coff;
    DBuf<int2> pq;
    pcnt.resize(nv);
    k_va_sort<<<g1(nv), 256, 0, s>>>(nv, kc, vptr, vlist, agg, ppos, plan.vlist2.p, plan.vpos.p, pcnt.p);
    MG_LAUNCH_CHECK();
    vpp.resize((size_t)nv + 1);
    scan_exclusive<int32_t>(pcnt.p, vpp.p, nv, s);
    plan.npairs = read_scalar(vpp.p + nv, s);
    plan.pstart.resize(plan.npairs + 1);
    pagg.resize(plan.npairs);
    ccnt.resize(nv);
    k_va_pairs<<<g1(nv), 256, 0, s>>>(nv, kc, vptr, plan.vlist2.p, agg, vpp.p, plan.pstart.p, pagg.p, ccnt.p);
    MG_LAUNCH_CHECK();
    const int32_t ninc32 = (int32_t)ninc;
    MG_CK(cudaMemcpyAsync(plan.pstart.p + plan.npairs, &ninc32, sizeof(int32_t), cudaMemcpyHostToDevice, s));
    coff.resize((size_t)nv + 1);
    scan_exclusive<int32_t>(ccnt.p, coff.p, nv, s);
    plan.ncontrib = read_scalar(coff.p + nv, s);
    key.resize(plan.ncontrib);
    pq.resize(plan.ncontrib);
    DBuf<int32_t> bad;
    bad.resize(1);
    MG_CK(cudaMemsetAsync(bad.p, 0, sizeof(int32_t), s));
    k_va_contrib<<<g1(nv), 256, 0, s>>>(nv, vpp.p, coff.p, pagg.p, crowptr, ccol, key.p, pq.p, bad.p);
    MG_LAUNCH_CHECK();
    if (read_scalar(bad.p, s)) throw Error(-1, "va_symbolic: product outside the coarse pattern");
    group_by_key(key.p, plan.ncontrib, cnnz, plan.cptr, clist, cnt, s, true);
    plan.cpq.resize(plan.ncontrib);
    k_va_permute<<<g1(plan.ncontrib), 256, 0, s>>>(plan.ncontrib, clist.p, pq.p, plan.cpq.p);
    MG_LAUNCH_CHECK();
    if (plan.ncontrib >= INT32_MAX) throw Error(-1, "va_symbolic: more than 2^31 products");
    plan.crange.resize(cnnz);
    k_va_crange<<<g1(n_agg), 256, 0, s>>>(n_agg, crowptr, plan.cptr.p, plan.crange.p);
    MG_LAUNCH_CHECK();
    plan.G.resize((size_t)plan.npairs * 4 * sizeof(double));  // either hot type (allocated outside capture)
    MG_CK(cudaStreamSynchronize(s));  // temporaries are freed on return
}

template <class T>
void va_numeric(VaPlan& plan, int kc, const T* h, const T* hv, const T* P, const int64_t* mptr,
                const int32_t* mlist, const T* at, int32_t n_agg, const int64_t* crowptr, T* cval, T* cdinv,
                cudaStream_t s) {
    G4<T>* G = reinterpret_cast<G4<T>*>(plan.G.p);
    if (plan.npairs) {
#define MG_VAG(KC, HV)                                                                                      \
    k_va_g<T, KC, HV><<<g1(plan.npairs), 256, 0, s>>>(plan.npairs, plan.pstart.p, plan.vlist2.p, plan.vpos.p, h, \
                                                      hv, plan.hv_stride, P, G)
        if (kc == 4) { if (hv) MG_VAG(4, true); else MG_VAG(4, false); }
        else { if (hv) MG_VAG(2, true); else MG_VAG(2, false); }
#undef MG_VAG
        MG_LAUNCH_CHECK();
    }
    k_va_a1<T><<<g1(plan.cnnz), 256, 0, s>>>(plan.cnnz, plan.crange.p, plan.cpq.p, G, cval);
    MG_LAUNCH_CHECK();
    if (n_agg) {
        k_va_a1_diag<T><<<(int)std::min<int64_t>(((int64_t)n_agg * 32 + 255) / 256, 148 * 16), 256, 0, s>>>(
            n_agg, plan.cptr.p, plan.cpq.p, G, crowptr, mptr, mlist, P, at, cval, cdinv);
        MG_LAUNCH_CHECK();
    }
}

template void va_numeric<float>(VaPlan&, int, const float*, const float*, const float*, const int64_t*, const int32_t*,
                                const float*, int32_t, const int64_t*, float*, float*, cudaStream_t);
template void va_numeric<double>(VaPlan&, int, const double*, const double*, const double*, const int64_t*, const int32_t*,
                                 const double*, int32_t, const int64_t*, double*, double*, cudaStream_t);

}  // namespace mgpbd
