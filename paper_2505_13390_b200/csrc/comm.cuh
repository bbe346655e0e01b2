// Communication layer of the row-partitioned (world > 1) MGPBD frame.
//
// Level 0 is split into contiguous row blocks balanced by nonzeros; every rank keeps full-length
// level-0 vectors indexed globally, owns rows [r0, r1) and receives a halo of the x entries its rows
// reference (the mesh order makes that two contiguous ranges).  Coarse levels and the setup are
// replicated (deterministic, so every rank builds the same hierarchy).  Collectives:
//   halo(v)        before every level-0 matrix pass        (send/recv with the owning ranks)
//   allreduce(x)   PCG dots, level-1 restriction, level-1 Galerkin values, dlambda
// Two backends: NCCL (one process per GPU) and "virtual ranks" (W contexts in one process on one
// GPU, host-synchronised; used by the tests to run the partitioned path on a single device).
#pragma once
#include <cuda_runtime.h>

#include <memory>
#include <vector>

#include "common.cuh"

namespace mgpbd {

struct Range {
    int32_t a = 0, b = 0;  // [a, b)
    int32_t size() const { return b > a ? b - a : 0; }
};

// Host-only partition logic (pure functions; exported through the C-ABI for CPU tests).
// rows split so each rank gets ~nnz/world nonzeros: r[p] = first row whose rowptr >= p*nnz/world.
std::vector<int32_t> partition_rows(const int64_t* rowptr, int32_t n, int world);
// For rank q with rows [r0,r1) referencing columns [minc, maxc]: the range it receives from each peer.
// recv[q][p] = columns owned by p inside q's referenced window (empty for p == q); rank p sends
// exactly recv[q][p] to q.
std::vector<std::vector<Range>> halo_plan(const std::vector<int32_t>& bounds, const std::vector<int32_t>& minc,
                                          const std::vector<int32_t>& maxc);

class Comm {
   public:
    virtual ~Comm() = default;
    virtual int rank() const = 0;
    virtual int world() const = 0;
    // in-place sum over ranks of a device buffer (double or float), stream-ordered
    virtual void allreduce(double* d, size_t n, cudaStream_t s) = 0;
    virtual void allreduce(float* d, size_t n, cudaStream_t s) = 0;
    // exchange: for each peer, send [ptr+send.a, ptr+send.b) and receive into [ptr+recv.a, ...)
    struct Xfer { int peer; Range send, recv; };
    virtual void exchange(void* base, size_t elem, const std::vector<Xfer>& xs, cudaStream_t s) = 0;
    // every rank's block [bounds[r], bounds[r+1]) of a full-length buffer replaces the others' copies
    // (variable-size allgather in place: one broadcast per root in a group)
    virtual void allgather_blocks(void* base, size_t elem, const std::vector<int32_t>& bounds, cudaStream_t s) = 0;
    virtual bool graph_capturable() const = 0;
};

// NCCL backend: id = 128-byte ncclUniqueId shared by all ranks (rank 0 creates it).
std::unique_ptr<Comm> make_nccl_comm(const void* id, int rank, int world, int device);
void nccl_unique_id(void* out128);

// Virtual-ranks backend: a group object shared by W contexts of one process (one thread each).
struct VirtualGroup;
VirtualGroup* vgroup_create(int world);
void vgroup_destroy(VirtualGroup* g);
std::unique_ptr<Comm> make_virtual_comm(VirtualGroup* g, int rank);

}  // namespace mgpbd
