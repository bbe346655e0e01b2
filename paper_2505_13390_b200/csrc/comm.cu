// Communication layer: row partition, halo plan, NCCL and virtual-ranks backends (see comm.cuh).
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>

#include "comm.cuh"

namespace mgpbd {

std::vector<int32_t> partition_rows(const int64_t* rowptr, int32_t n, int world) {
    std::vector<int32_t> b(world + 1, 0);
    const int64_t nnz = rowptr[n];
    for (int p = 1; p < world; ++p) {
        const int64_t target = (nnz * p) / world;
        b[p] = (int32_t)(std::lower_bound(rowptr, rowptr + n + 1, target) - rowptr);
        if (b[p] < b[p - 1]) b[p] = b[p - 1];
        if (b[p] > n) b[p] = n;
    }
    b[world] = n;
    return b;
}

std::vector<std::vector<Range>> halo_plan(const std::vector<int32_t>& bounds, const std::vector<int32_t>& minc,
                                          const std::vector<int32_t>& maxc) {
    const int W = (int)bounds.size() - 1;
    std::vector<std::vector<Range>> recv(W, std::vector<Range>(W));
    for (int q = 0; q < W; ++q) {
        if (bounds[q + 1] <= bounds[q]) continue;  // empty rank references nothing
        for (int p = 0; p < W; ++p) {
            if (p == q) continue;
            Range r;
            r.a = std::max(minc[q], bounds[p]);
            r.b = std::min(maxc[q] + 1, bounds[p + 1]);
            if (r.b > r.a) recv[q][p] = r;
        }
    }
    return recv;
}

// ----------------------------------------------------------------------------- NCCL
#define MG_NCCL(call)                                                                              \
    do {                                                                                           \
        ncclResult_t r_ = (call);                                                                  \
        if (r_ != ncclSuccess)                                                                     \
            throw ::mgpbd::Error(-3, std::string(#call) + ": " + ncclGetErrorString(r_));          \
    } while (0)

class NcclComm : public Comm {
   public:
    NcclComm(const void* id, int rank, int world, int device) : r_(rank), w_(world) {
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        MG_CK(cudaSetDevice(device));
        MG_NCCL(ncclCommInitRank(&comm_, world, uid, rank));
    }
    ~NcclComm() override { if (comm_) ncclCommDestroy(comm_); }
    int rank() const override { return r_; }
    int world() const override { return w_; }
    void allreduce(double* d, size_t n, cudaStream_t s) override {
        if (n) MG_NCCL(ncclAllReduce(d, d, n, ncclFloat64, ncclSum, comm_, s));
    }
    void allreduce(float* d, size_t n, cudaStream_t s) override {
        if (n) MG_NCCL(ncclAllReduce(d, d, n, ncclFloat32, ncclSum, comm_, s));
    }
    void exchange(void* base, size_t elem, const std::vector<Xfer>& xs, cudaStream_t s) override {
        if (xs.empty()) return;
        char* b = static_cast<char*>(base);
        MG_NCCL(ncclGroupStart());
        for (const Xfer& x : xs) {
            if (x.send.size()) MG_NCCL(ncclSend(b + (size_t)x.send.a * elem, (size_t)x.send.size() * elem, ncclUint8, x.peer, comm_, s));
            if (x.recv.size()) MG_NCCL(ncclRecv(b + (size_t)x.recv.a * elem, (size_t)x.recv.size() * elem, ncclUint8, x.peer, comm_, s));
        }
        MG_NCCL(ncclGroupEnd());
    }
    void allgather_blocks(void* base, size_t elem, const std::vector<int32_t>& bounds, cudaStream_t s) override {
        char* b = static_cast<char*>(base);
        MG_NCCL(ncclGroupStart());
        for (int r = 0; r < w_; ++r) {
            const size_t n = (size_t)(bounds[r + 1] - bounds[r]) * elem;
            if (n) MG_NCCL(ncclBroadcast(b + (size_t)bounds[r] * elem, b + (size_t)bounds[r] * elem, n, ncclUint8, r, comm_, s));
        }
        MG_NCCL(ncclGroupEnd());
    }
    bool graph_capturable() const override { return true; }

   private:
    ncclComm_t comm_ = nullptr;
    int r_, w_;
};

std::unique_ptr<Comm> make_nccl_comm(const void* id, int rank, int world, int device) {
    return std::unique_ptr<Comm>(new NcclComm(id, rank, world, device));
}
void nccl_unique_id(void* out128) {
    ncclUniqueId uid;
    MG_NCCL(ncclGetUniqueId(&uid));
    std::memcpy(out128, &uid, sizeof(uid));
}

// ----------------------------------------------------------------------------- virtual ranks
struct VirtualGroup {
    int world;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t generation = 0;
    std::vector<void*> ptr;
    explicit VirtualGroup(int w) : world(w), ptr(w, nullptr) {}
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const uint64_t gen = generation;
        if (++arrived == world) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen; });
        }
    }
};

VirtualGroup* vgroup_create(int world) { return new VirtualGroup(world); }
void vgroup_destroy(VirtualGroup* g) { delete g; }

namespace {
template <class T>
struct Ptrs { const T* p[8]; };
template <class T>
__global__ void k_vsum(size_t n, int w, Ptrs<T> in, T* __restrict__ out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        T s = in.p[0][i];
        for (int q = 1; q < w; ++q) s += in.p[q][i];  // fixed rank order
        out[i] = s;
    }
}
}  // namespace

class VirtualComm : public Comm {
   public:
    VirtualComm(VirtualGroup* g, int rank) : g_(g), r_(rank) {
        if (g->world > 8) throw Error(-1, "virtual ranks: world <= 8");
    }
    int rank() const override { return r_; }
    int world() const override { return g_->world; }
    void allreduce(double* d, size_t n, cudaStream_t s) override { sum<double>(d, n, s); }
    void allreduce(float* d, size_t n, cudaStream_t s) override { sum<float>(d, n, s); }
    void exchange(void* base, size_t elem, const std::vector<Xfer>& xs, cudaStream_t s) override {
        MG_CK(cudaStreamSynchronize(s));
        g_->ptr[r_] = base;
        g_->barrier();
        for (const Xfer& x : xs)
            if (x.recv.size())
                MG_CK(cudaMemcpyAsync(static_cast<char*>(base) + (size_t)x.recv.a * elem,
                                      static_cast<const char*>(g_->ptr[x.peer]) + (size_t)x.recv.a * elem,
                                      (size_t)x.recv.size() * elem, cudaMemcpyDeviceToDevice, s));
        MG_CK(cudaStreamSynchronize(s));
        g_->barrier();
    }
    void allgather_blocks(void* base, size_t elem, const std::vector<int32_t>& bounds, cudaStream_t s) override {
        MG_CK(cudaStreamSynchronize(s));
        g_->ptr[r_] = base;
        g_->barrier();
        for (int q = 0; q < g_->world; ++q) {
            const size_t n = (size_t)(bounds[q + 1] - bounds[q]) * elem;
            if (q != r_ && n)
                MG_CK(cudaMemcpyAsync(static_cast<char*>(base) + (size_t)bounds[q] * elem,
                                      static_cast<const char*>(g_->ptr[q]) + (size_t)bounds[q] * elem, n,
                                      cudaMemcpyDeviceToDevice, s));
        }
        MG_CK(cudaStreamSynchronize(s));
        g_->barrier();
    }
    bool graph_capturable() const override { return false; }

   private:
    template <class T>
    void sum(T* d, size_t n, cudaStream_t s) {
        if (!n) return;
        tmp_.resize(n * sizeof(T));
        MG_CK(cudaStreamSynchronize(s));
        g_->ptr[r_] = d;
        g_->barrier();
        Ptrs<T> in{};
        for (int q = 0; q < g_->world; ++q) in.p[q] = static_cast<const T*>(g_->ptr[q]);
        k_vsum<T><<<(int)std::min<size_t>((n + 255) / 256, 148 * 8), 256, 0, s>>>(n, g_->world, in,
                                                                                  reinterpret_cast<T*>(tmp_.p));
        MG_LAUNCH_CHECK();
        MG_CK(cudaStreamSynchronize(s));
        g_->barrier();  // every rank has read every input
        MG_CK(cudaMemcpyAsync(d, tmp_.p, n * sizeof(T), cudaMemcpyDeviceToDevice, s));
    }
    VirtualGroup* g_;
    int r_;
    DBuf<unsigned char> tmp_;
};

std::unique_ptr<Comm> make_virtual_comm(VirtualGroup* g, int rank) {
    return std::unique_ptr<Comm>(new VirtualComm(g, rank));
}

}  // namespace mgpbd
