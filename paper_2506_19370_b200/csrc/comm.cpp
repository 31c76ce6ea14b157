// Transports of the multi-GPU superstep (see comm.h).
#include "comm.h"

#include <atomic>
#include <cstdint>
#include <cstring>
#include <algorithm>
#include <cstdio>
#include <random>
#include <type_traits>

#include "fc_tables.h"  // Error
#include "fcsg_common.h"

#if defined(FCSG_EMULATE)
#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <unistd.h>
#else
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#endif

namespace fcsg {

#if !defined(FCSG_EMULATE)
// ---------------------------------------------------------------------------
// NCCL (CUDA build)

namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static bool loaded = false;
    if (loaded) return api;
    // the process's NCCL if one is loaded (torch's), else the system library
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw Error(kConfig, std::string("multi-GPU: libnccl.so.2 not found: ") + dlerror());
    auto sym = [&](auto& fn, const char* name) {
        fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
        if (!fn) throw Error(kConfig, std::string("multi-GPU: NCCL symbol missing: ") + name);
    };
    sym(api.get_unique_id, "ncclGetUniqueId");
    sym(api.comm_init_rank, "ncclCommInitRank");
    sym(api.comm_destroy, "ncclCommDestroy");
    sym(api.group_start, "ncclGroupStart");
    sym(api.group_end, "ncclGroupEnd");
    sym(api.send, "ncclSend");
    sym(api.recv, "ncclRecv");
    sym(api.all_reduce, "ncclAllReduce");
    sym(api.error_string, "ncclGetErrorString");
    loaded = true;
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw Error(kCuda, std::string(what) + ": " + nccl().error_string(r));
}

class NcclComm : public Comm {
  public:
    NcclComm(int nranks, int rank, const char id[kCommIdBytes]) {
        static_assert(sizeof(ncclUniqueId) == kCommIdBytes, "ncclUniqueId size");
        rank_ = rank;
        size_ = nranks;
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        nccl_check(nccl().comm_init_rank(&comm_, nranks, uid, rank), "ncclCommInitRank");
    }
    ~NcclComm() override {
        if (comm_) nccl().comm_destroy(comm_);
    }
    void group_start() override {
        ops_.clear();
    }
    void send(const double* buf, size_t count, int peer) override { ops_.push_back({true, const_cast<double*>(buf), count, peer}); }
    void recv(double* buf, size_t count, int peer) override { ops_.push_back({false, buf, count, peer}); }
    void group_end(void* stream) override {
        if (ops_.empty()) return;
        const auto s = static_cast<cudaStream_t>(stream);
        nccl_check(nccl().group_start(), "ncclGroupStart");
        for (const Op& o : ops_) {
            if (o.count == 0) continue;
            if (o.is_send) nccl_check(nccl().send(o.buf, o.count, ncclFloat64, o.peer, comm_, s), "ncclSend");
            else nccl_check(nccl().recv(o.buf, o.count, ncclFloat64, o.peer, comm_, s), "ncclRecv");
        }
        nccl_check(nccl().group_end(), "ncclGroupEnd");
        ops_.clear();
    }
    void allreduce_min_u64(unsigned long long* p, void* stream) override {
        nccl_check(nccl().all_reduce(p, p, 1, ncclUint64, ncclMin, comm_, static_cast<cudaStream_t>(stream)),
                   "ncclAllReduce");
    }

  private:
    struct Op {
        bool is_send;
        double* buf;
        size_t count;
        int peer;
    };
    ncclComm_t comm_ = nullptr;
    std::vector<Op> ops_;
};

}  // namespace

void comm_unique_id(char id[kCommIdBytes]) {
    ncclUniqueId uid;
    nccl_check(nccl().get_unique_id(&uid), "ncclGetUniqueId");
    std::memcpy(id, &uid, sizeof(uid));
}

std::unique_ptr<Comm> comm_create(int nranks, int rank, const char id[kCommIdBytes]) {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw Error(kUsage, "bad rank / world size");
    return std::make_unique<NcclComm>(nranks, rank, id);
}

#else
// ---------------------------------------------------------------------------
// Shared-memory mailboxes (emulation build; TEST HARNESS for the CPU
// world-size-2 tests). Box (a, b) carries a's messages to b in chunks of
// kCap bytes: the sender waits for the previous chunk's ack, writes, bumps
// seq; the receiver waits for seq, reads, bumps ack. group_end progresses
// every queued send and recv together, so two ranks sending each other
// multi-chunk messages cannot deadlock.

namespace {

constexpr size_t kCap = 1 << 20;
struct alignas(64) Box {
    std::atomic<uint64_t> seq;
    std::atomic<uint64_t> ack;
    uint64_t bytes;
    char pad[40];
    char data[kCap];
};

class ShmComm : public Comm {
  public:
    ShmComm(int nranks, int rank, const char id[kCommIdBytes]) {
        rank_ = rank;
        size_ = nranks;
        name_.assign(id, strnlen(id, kCommIdBytes));
        bytes_ = sizeof(Box) * static_cast<size_t>(nranks) * nranks;
        const int fd = shm_open(name_.c_str(), O_CREAT | O_RDWR, 0600);
        if (fd < 0) throw Error(kOther, "shm_open failed: " + name_);
        if (ftruncate(fd, static_cast<off_t>(bytes_)) != 0) {
            close(fd);
            throw Error(kOther, "ftruncate failed: " + name_);
        }
        void* p = mmap(nullptr, bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        close(fd);
        if (p == MAP_FAILED) throw Error(kOther, "mmap failed: " + name_);
        boxes_ = static_cast<Box*>(p);
    }
    ~ShmComm() override {
        munmap(boxes_, bytes_);
        shm_unlink(name_.c_str());  // the other ranks keep their mappings
    }
    void group_start() override { ops_.clear(); }
    void send(const double* buf, size_t count, int peer) override {
        ops_.push_back({true, reinterpret_cast<char*>(const_cast<double*>(buf)), count * sizeof(double), peer, 0});
    }
    void recv(double* buf, size_t count, int peer) override {
        ops_.push_back({false, reinterpret_cast<char*>(buf), count * sizeof(double), peer, 0});
    }
    void group_end(void*) override {
        // empty transfers are skipped on both sides (the counts agree)
        bool pending = true;
        while (pending) {
            pending = false;
            bool moved = false;
            for (Op& o : ops_) {
                if (o.done >= o.bytes) continue;
                if (o.is_send) {
                    Box& b = box(rank_, o.peer);
                    if (b.ack.load(std::memory_order_acquire) == b.seq.load(std::memory_order_relaxed)) {
                        const size_t n = std::min(kCap, o.bytes - o.done);
                        std::memcpy(b.data, o.buf + o.done, n);
                        b.bytes = n;
                        b.seq.fetch_add(1, std::memory_order_release);
                        o.done += n;
                        moved = true;
                    }
                } else {
                    Box& b = box(o.peer, rank_);
                    if (b.seq.load(std::memory_order_acquire) != b.ack.load(std::memory_order_relaxed)) {
                        const size_t n = b.bytes;
                        if (o.done + n > o.bytes) throw Error(kUsage, "shm comm: message longer than the receive");
                        std::memcpy(o.buf + o.done, b.data, n);
                        b.ack.fetch_add(1, std::memory_order_release);
                        o.done += n;
                        moved = true;
                    }
                }
                if (o.done < o.bytes) pending = true;
            }
            if (pending && !moved) sched_yield();
        }
        ops_.clear();
    }
    void allreduce_min_u64(unsigned long long* p, void*) override {
        std::vector<unsigned long long> in(size_);
        const double* mine = reinterpret_cast<const double*>(p);
        group_start();
        for (int r = 0; r < size_; ++r)
            if (r != rank_) {
                send(mine, 1, r);
                recv(reinterpret_cast<double*>(&in[r]), 1, r);
            }
        group_end(nullptr);
        for (int r = 0; r < size_; ++r)
            if (r != rank_ && in[r] < *p) *p = in[r];
    }

  private:
    struct Op {
        bool is_send;
        char* buf;
        size_t bytes;
        int peer;
        size_t done;
    };
    Box& box(int from, int to) { return boxes_[static_cast<size_t>(from) * size_ + to]; }
    std::string name_;
    size_t bytes_ = 0;
    Box* boxes_ = nullptr;
    std::vector<Op> ops_;
};

}  // namespace

void comm_unique_id(char id[kCommIdBytes]) {
    std::random_device rd;
    std::memset(id, 0, kCommIdBytes);
    std::snprintf(id, kCommIdBytes, "/fcsg_comm_%08x%08x", rd(), rd());
}

std::unique_ptr<Comm> comm_create(int nranks, int rank, const char id[kCommIdBytes]) {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw Error(kUsage, "bad rank / world size");
    return std::make_unique<ShmComm>(nranks, rank, id);
}
#endif

}  // namespace fcsg
