// Dense operator of the bottom of the V-cycle (reading c27), see subcycle.cuh.
#include <algorithm>

#include "subcycle.cuh"
#include "util.cuh"

namespace mgpbd {

namespace {

constexpr int SB = 256;   // threads per CTA
constexpr int CB = 4;     // unit-vector columns per CTA pass

// One thread per (row, column) pair: column cc = t % CB, rows t / CB + k SB / CB.  Vectors are stored
// row-interleaved (element (i, cc) at i CB + cc), so the CB threads of a row read consecutive words and
// load the same CSR entries (broadcast).
template <class T>
__global__ void __launch_bounds__(SB) k_subcycle_matrix(const __grid_constant__ SubCycle<T> c, double* __restrict__ M) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* sm = reinterpret_cast<T*>(smem_raw);
    constexpr int RS = SB / CB;
    const int t = threadIdx.x, cc = t % CB, rt = t / CB;
    const int32_t n0 = c.L[0].n;
    const int nu = c.nu;
    T* buf[3] = {sm + c.o_s0, sm + c.o_s1, sm + c.o_s2};
    // (A x)_i of level L for this thread's column
    auto rowsum = [&](const SubLevel<T>& L, const T* x, int32_t i) {
        double s = 0.0;
        for (int64_t e = L.rowptr[i]; e < L.rowptr[i + 1]; ++e) s += (double)L.val[e] * (double)x[(int64_t)L.col[e] * CB + cc];
        return s;
    };
    // x_out = x + om D^-1 (b - A x) + al (x - xprev), xprev == nullptr: 0 (the hot cycle's step)
    auto step = [&](const SubLevel<T>& L, const T* b, const T* x, const T* xprev, double om, double al, T* out) {
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
            const SubLevel<T>& L = c.L[k];
            const T* b = sm + L.o_b;
            T* xs = sm + L.o_xs;
            int cur = 0, prv = -1;
            for (int32_t i = rt; i < L.n; i += RS)  // step 0 from x = 0
                buf[0][i * CB + cc] = (T)(L.om[0] * (double)L.dinv[i] * (double)b[i * CB + cc]);
            __syncthreads();
            for (int s = 1; s < nu; ++s) {
                const int nxt = (prv < 0) ? (cur + 1) % 3 : 3 - cur - prv;
                step(L, b, buf[cur], prv < 0 ? nullptr : buf[prv], L.om[s], L.al[s], buf[nxt]);
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
            const SubLevel<T>& C = c.L[k + 1];
            T* bc = sm + C.o_b;
            for (int32_t a = rt; a < C.n; a += RS) {  // members ascending (the hot restriction's order)
                double s = 0.0;
                for (int64_t e = L.mptr[a]; e < L.mptr[a + 1]; ++e) s += (double)buf[rb][(int64_t)L.mlist[e] * CB + cc];
                bc[a * CB + cc] = (T)s;
            }
            __syncthreads();
        }
        // ---- coarsest: z = Ainv b
        int zb = 0;
        {
            const SubLevel<T>& C = c.L[c.K - 1];
            const T* b = sm + C.o_b;
            for (int32_t i = rt; i < C.n; i += RS) {
                double s = 0.0;
                const double* Ai = c.Ainv + (int64_t)i * C.n;
                for (int32_t j = 0; j < C.n; ++j) s += Ai[j] * (double)b[j * CB + cc];
                buf[zb][i * CB + cc] = (T)s;
            }
            __syncthreads();
        }
        // ---- up: x = xs + P z_c[agg], nu smoothing steps
        for (int k = c.K - 2; k >= 0; --k) {
            const SubLevel<T>& L = c.L[k];
            const T* b = sm + L.o_b;
            const T* xs = sm + L.o_xs;
            const T* zc = buf[zb];
            int cur = (zb + 1) % 3, prv = -1;
            for (int32_t i = rt; i < L.n; i += RS)
                buf[cur][i * CB + cc] = (T)((double)xs[i * CB + cc] + (double)L.P[i] * (double)zc[(int64_t)L.agg[i] * CB + cc]);
            __syncthreads();
            for (int s = 0; s < nu; ++s) {
                const int nxt = (prv < 0) ? (cur + 1) % 3 : 3 - cur - prv;
                step(L, b, buf[cur], prv < 0 ? nullptr : buf[prv], L.om[s], L.al[s], buf[nxt]);
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
    const uint64_t bytes = (uint64_t)off * sizeof(T);
    if (bytes > cap) return false;
    c.smem = (uint32_t)bytes;
    return try_raise_dyn_smem((const void*)k_subcycle_matrix<T>, c.smem);
}

template <class T>
void subcycle_matrix(const SubCycle<T>& c, double* M, cudaStream_t s) {
    const int32_t n0 = c.L[0].n;
    if (!n0) return;
    int dev = 0, sms = 148, occ = 1;
    MG_CK(cudaGetDevice(&dev));
    MG_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    MG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_subcycle_matrix<T>, SB, c.smem));
    const int blocks = (n0 + CB - 1) / CB;
    const int g = std::max(1, std::min(blocks, sms * std::max(occ, 1)));
    k_subcycle_matrix<T><<<g, SB, c.smem, s>>>(c, M);
    MG_LAUNCH_CHECK();
}

template bool subcycle_plan<float>(SubCycle<float>&, uint32_t);
template bool subcycle_plan<double>(SubCycle<double>&, uint32_t);
template void subcycle_matrix<float>(const SubCycle<float>&, double*, cudaStream_t);
template void subcycle_matrix<double>(const SubCycle<double>&, double*, cudaStream_t);

}  // namespace mgpbd
