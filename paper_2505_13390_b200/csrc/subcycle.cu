// Dense operator of the bottom of the V-cycle (reading c27), see subcycle.cuh.
#include <algorithm>

#include "subcycle.cuh"
#include "util.cuh"

namespace mgpbd {

namespace {

#ifndef MGPBD_SUB_SB
#define MGPBD_SUB_SB 512
#endif
#ifndef MGPBD_SUB_CB
#define MGPBD_SUB_CB 4
#endif
constexpr int SB = MGPBD_SUB_SB;   // threads per CTA
constexpr int CB = MGPBD_SUB_CB;   // unit-vector columns per CTA pass

// Level data as the kernel reads it: staged in shared memory (32-bit offsets) or in global memory.
template <class T, bool ST>
struct LvView {
    int32_t n;
    const void* rp;   // int32 (staged) / int64 row offsets
    const int32_t* col;
    const T* val;
    const T* dinv;
    const T* P;
    const int32_t* agg;
    const void* mp;   // int32 (staged) / int64 member offsets
    const int32_t* ml;
    __device__ __forceinline__ int64_t rb(int32_t i) const {
        return ST ? (int64_t) static_cast<const int32_t*>(rp)[i] : static_cast<const int64_t*>(rp)[i];
    }
    __device__ __forceinline__ int64_t mb(int32_t a) const {
        return ST ? (int64_t) static_cast<const int32_t*>(mp)[a] : static_cast<const int64_t*>(mp)[a];
    }
};

// One thread per (row, column) pair: column cc = t % CB, rows t / CB + k SB / CB.  Vectors are stored
// row-interleaved (element (i, cc) at i CB + cc), so the CB threads of a row read consecutive words and
// load the same CSR entries (broadcast).  ST: the level data and Ainv are first copied into shared memory
// (once per CTA; every column block then reads them at shared-memory latency).
template <class T, bool ST>
__global__ void __launch_bounds__(SB) k_subcycle_matrix(const __grid_constant__ SubCycle<T> c, double* __restrict__ M) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* sm = reinterpret_cast<T*>(smem_raw);
    constexpr int RS = SB / CB;
    const int t = threadIdx.x, cc = t % CB, rt = t / CB;
    const int32_t n0 = c.L[0].n;
    const int nu = c.nu;
    LvView<T, ST> V[SUB_MAXL];
    const double* Ainv = c.Ainv;
    for (int k = 0; k < c.K; ++k) {
        const SubLevel<T>& L = c.L[k];
        const bool last = k + 1 == c.K;
        if (ST) {
            unsigned char* b = smem_raw;
            int32_t* rp = reinterpret_cast<int32_t*>(b + L.s_rp);
            int32_t* col = reinterpret_cast<int32_t*>(b + L.s_col);
            T* val = reinterpret_cast<T*>(b + L.s_val);
            T* dinv = reinterpret_cast<T*>(b + L.s_dinv);
            for (int32_t i = t; i <= L.n; i += SB) rp[i] = (int32_t)L.rowptr[i];
            for (int32_t e = t; e < L.nnz; e += SB) { col[e] = L.col[e]; val[e] = L.val[e]; }
            for (int32_t i = t; i < L.n; i += SB) dinv[i] = L.dinv[i];
            V[k] = {L.n, rp, col, val, dinv, nullptr, nullptr, nullptr, nullptr};
            if (!last) {
                T* P = reinterpret_cast<T*>(b + L.s_P);
                int32_t* agg = reinterpret_cast<int32_t*>(b + L.s_agg);
                int32_t* mp = reinterpret_cast<int32_t*>(b + L.s_mp);
                int32_t* ml = reinterpret_cast<int32_t*>(b + L.s_ml);
                for (int32_t i = t; i < L.n; i += SB) { P[i] = L.P[i]; agg[i] = L.agg[i]; ml[i] = L.mlist[i]; }
                for (int32_t a = t; a <= L.n_next; a += SB) mp[a] = (int32_t)L.mptr[a];
                V[k].P = P; V[k].agg = agg; V[k].mp = mp; V[k].ml = ml;
            }
        } else {
            V[k] = {L.n, L.rowptr, L.col, L.val, L.dinv, L.P, L.agg, L.mptr, L.mlist};
        }
    }
    if (ST) {
        const int32_t nc = c.L[c.K - 1].n;
        double* A = reinterpret_cast<double*>(smem_raw + c.s_ainv);
        for (int64_t e = t; e < (int64_t)nc * nc; e += SB) A[e] = c.Ainv[e];
        Ainv = A;
        __syncthreads();
    }
    T* buf[3] = {sm + c.o_s0, sm + c.o_s1, sm + c.o_s2};
    // (A x)_i of level L for this thread's column
    auto rowsum = [&](const LvView<T, ST>& L, const T* x, int32_t i) {
        double s = 0.0;
        const int64_t e1 = L.rb(i + 1);
        for (int64_t e = L.rb(i); e < e1; ++e) s += (double)L.val[e] * (double)x[(int64_t)L.col[e] * CB + cc];
        return s;
    };
    // x_out = x + om D^-1 (b - A x) + al (x - xprev), xprev == nullptr: 0 (the hot cycle's step)
    auto step = [&](const LvView<T, ST>& L, const T* b, const T* x, const T* xprev, double om, double al, T* out) {
        for (int32_t i = rt; i < L.n; i += RS) {
            const double xi = (double)x[i * CB + cc];
            double y = xi + om * (double)L.dinv[i] * ((double)b[i * CB + cc] - rowsum(L, x, i));
            if (al != 0.0) y += al * (xi - (xprev ? (double)xprev[i * CB + cc] : 0.0));
            out[i * CB + cc] = (T)y;
        }
        __syncthreads();
    };
    for (int32_t jb = blockIdx.x * CB; jb < n0; jb += gridDim.x * CB) {
        {   // b_0 = e_{jb + cc}
            T* b0 = sm + c.L[0].o_b;
            for (int32_t i = rt; i < n0; i += RS) b0[i * CB + cc] = i == jb + cc ? (T)1 : (T)0;
            __syncthreads();
        }
        // ---- down: nu smoothing steps from x = 0, residual, restriction
        for (int k = 0; k + 1 < c.K; ++k) {
            const SubLevel<T>& Ls = c.L[k];
            const LvView<T, ST>& L = V[k];
            const T* b = sm + Ls.o_b;
            T* xs = sm + Ls.o_xs;
            int cur = 0, prv = -1;
            for (int32_t i = rt; i < L.n; i += RS)  // step 0 from x = 0
                buf[0][i * CB + cc] = (T)(Ls.om[0] * (double)L.dinv[i] * (double)b[i * CB + cc]);
            __syncthreads();
            for (int s = 1; s < nu; ++s) {
                const int nxt = (prv < 0) ? (cur + 1) % 3 : 3 - cur - prv;
                step(L, b, buf[cur], prv < 0 ? nullptr : buf[prv], Ls.om[s], Ls.al[s], buf[nxt]);
                prv = cur;
                cur = nxt;
            }
            const int rb = (cur + 1) % 3;  // residual times P (the restriction input)
            for (int32_t i = rt; i < L.n; i += RS) {
                const T xi = buf[cur][i * CB + cc];
                xs[i * CB + cc] = xi;
                buf[rb][i * CB + cc] = (T)((double)L.P[i] * ((double)b[i * CB + cc] - rowsum(L, buf[cur], i)));
            }
            __syncthreads();
            T* bc = sm + c.L[k + 1].o_b;
            for (int32_t a = rt; a < V[k + 1].n; a += RS) {  // members ascending (the hot restriction's order)
                double s = 0.0;
                const int64_t m1 = L.mb(a + 1);
                for (int64_t e = L.mb(a); e < m1; ++e) s += (double)buf[rb][(int64_t)L.ml[e] * CB + cc];
                bc[a * CB + cc] = (T)s;
            }
            __syncthreads();
        }
        // ---- coarsest: z = Ainv b
        int zb = 0;
        {
            const int32_t nc = V[c.K - 1].n;
            const T* b = sm + c.L[c.K - 1].o_b;
            for (int32_t i = rt; i < nc; i += RS) {
                double s = 0.0;
                const double* Ai = Ainv + (int64_t)i * nc;
                for (int32_t j = 0; j < nc; ++j) s += Ai[j] * (double)b[j * CB + cc];
                buf[zb][i * CB + cc] = (T)s;
            }
            __syncthreads();
        }
        // ---- up: x = xs + P z_c[agg], nu smoothing steps
        for (int k = c.K - 2; k >= 0; --k) {
            const SubLevel<T>& Ls = c.L[k];
            const LvView<T, ST>& L = V[k];
            const T* b = sm + Ls.o_b;
            const T* xs = sm + Ls.o_xs;
            const T* zc = buf[zb];
            int cur = (zb + 1) % 3, prv = -1;
            for (int32_t i = rt; i < L.n; i += RS)
                buf[cur][i * CB + cc] = (T)((double)xs[i * CB + cc] + (double)L.P[i] * (double)zc[(int64_t)L.agg[i] * CB + cc]);
            __syncthreads();
            for (int s = 0; s < nu; ++s) {
                const int nxt = (prv < 0) ? (cur + 1) % 3 : 3 - cur - prv;
                step(L, b, buf[cur], prv < 0 ? nullptr : buf[prv], Ls.om[s], Ls.al[s], buf[nxt]);
                prv = cur;
                cur = nxt;
            }
            zb = cur;
        }
        const int32_t j = jb + cc;
        if (j < n0)
            for (int32_t i = rt; i < n0; i += RS) M[(int64_t)i * n0 + j] = (double)buf[zb][i * CB + cc];
        __syncthreads();
    }
}

}  // namespace

template <class T>
bool subcycle_plan(SubCycle<T>& c, uint32_t cap) {
    if (c.K < 2 || c.K > SUB_MAXL) return false;
    uint32_t off = 0;
    int32_t nmax = 0;
    for (int k = 0; k < c.K; ++k) {
        SubLevel<T>& L = c.L[k];
        L.o_b = off;
        off += (uint32_t)L.n * CB;
        if (k + 1 < c.K) { L.o_xs = off; off += (uint32_t)L.n * CB; }
        nmax = std::max(nmax, L.n);
    }
    c.o_s0 = off; off += (uint32_t)nmax * CB;
    c.o_s1 = off; off += (uint32_t)nmax * CB;
    c.o_s2 = off; off += (uint32_t)nmax * CB;
    const uint64_t vbytes = ((uint64_t)off * sizeof(T) + 15) & ~(uint64_t)15;
    if (vbytes > cap) return false;
    c.vec_bytes = (uint32_t)vbytes;
    // staged layout behind the vectors (16-byte aligned sections)
    uint64_t b = vbytes;
    auto take = [&](uint64_t bytes) { const uint64_t o = b; b += (bytes + 15) & ~(uint64_t)15; return (uint32_t)o; };
    for (int k = 0; k < c.K; ++k) {
        SubLevel<T>& L = c.L[k];
        L.s_rp = take(4ull * (L.n + 1));
        L.s_col = take(4ull * L.nnz);
        L.s_val = take(sizeof(T) * (uint64_t)L.nnz);
        L.s_dinv = take(sizeof(T) * (uint64_t)L.n);
        if (k + 1 < c.K) {
            L.s_P = take(sizeof(T) * (uint64_t)L.n);
            L.s_agg = take(4ull * L.n);
            L.s_mp = take(4ull * (L.n_next + 1));
            L.s_ml = take(4ull * L.n);
        }
    }
    const uint64_t nc = (uint64_t)c.L[c.K - 1].n;
    c.s_ainv = take(8ull * nc * nc);
    c.staged = b <= cap;
    c.smem = c.staged ? (uint32_t)b : c.vec_bytes;
    const void* k = c.staged ? (const void*)k_subcycle_matrix<T, true> : (const void*)k_subcycle_matrix<T, false>;
    return try_raise_dyn_smem(k, c.smem);
}

template <class T>
void subcycle_matrix(const SubCycle<T>& c, double* M, cudaStream_t s) {
    const int32_t n0 = c.L[0].n;
    if (!n0) return;
    int dev = 0, sms = 148, occ = 1;
    MG_CK(cudaGetDevice(&dev));
    MG_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const void* k = c.staged ? (const void*)k_subcycle_matrix<T, true> : (const void*)k_subcycle_matrix<T, false>;
    MG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, SB, c.smem));
    const int blocks = (n0 + CB - 1) / CB;
    const int g = std::max(1, std::min(blocks, sms * std::max(occ, 1)));
    if (c.staged) k_subcycle_matrix<T, true><<<g, SB, c.smem, s>>>(c, M);
    else k_subcycle_matrix<T, false><<<g, SB, c.smem, s>>>(c, M);
    MG_LAUNCH_CHECK();
}

template bool subcycle_plan<float>(SubCycle<float>&, uint32_t);
template bool subcycle_plan<double>(SubCycle<double>&, uint32_t);
template void subcycle_matrix<float>(const SubCycle<float>&, double*, cudaStream_t);
template void subcycle_matrix<double>(const SubCycle<double>&, double*, cudaStream_t);

}  // namespace mgpbd
