// Device-ordered transport of the multi-GPU superstep.
//
// The reference exchanges fringe values between worker threads through
// shared memory behind barriers (src/runtime.cpp:433-454 phase 6, :352-371
// the viscosity blend's donor reads, :492-497 the dt minimum). Across GPUs
// each rank owns a block of subpatches and moves, per RK stage, only the
// packed donor values its neighbour ranks need, and per step the mu_hat
// values of the blend and one dt minimum.
//
// Comm is enqueued on the engine stream like a kernel -- no host
// synchronisation anywhere in a step -- so the whole multi-rank superstep is
// captured in one CUDA graph:
//  * NcclComm (CUDA build): grouped ncclSend / ncclRecv to the neighbour
//    ranks only, ncclAllReduce(MIN) of the dt bits; NVLink / NVSwitch P2P.
//    libnccl.so.2 is opened at run time (the copy torch already loaded when
//    it is in the process, else the system one), so the library has no link
//    dependency on NCCL.
//  * ShmComm (emulation build, TEST HARNESS): the same send / recv / min
//    semantics between CPU processes through a POSIX shared-memory mailbox
//    per ordered rank pair, so the world-size-2 CPU tests drive exactly the
//    engine code the GPU ranks run.
#pragma once

#include <cstddef>
#include <memory>
#include <string>
#include <vector>

namespace fcsg {

constexpr int kCommIdBytes = 128;  // sizeof(ncclUniqueId)

class Comm {
  public:
    virtual ~Comm() = default;
    int rank() const { return rank_; }
    int size() const { return size_; }
    // point-to-point transfers of one group: queued by send / recv, issued
    // together (NCCL: one ncclGroupStart / End, so the pairs cannot deadlock)
    virtual void group_start() = 0;
    virtual void send(const double* buf, size_t count, int peer) = 0;
    virtual void recv(double* buf, size_t count, int peer) = 0;
    virtual void group_end(void* stream) = 0;
    // in-place MIN all-reduce of one uint64 in device memory
    virtual void allreduce_min_u64(unsigned long long* p, void* stream) = 0;

  protected:
    int rank_ = 0, size_ = 1;
};

// a fresh rendezvous id (rank 0 creates it; the caller broadcasts it)
void comm_unique_id(char id[kCommIdBytes]);
// every rank calls this collectively with the same id
std::unique_ptr<Comm> comm_create(int nranks, int rank, const char id[kCommIdBytes]);

}  // namespace fcsg
